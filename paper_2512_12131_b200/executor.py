"""Device executor of one decoder block under a BTP plan, forward + backward, on one TP rank.

Follows the reference's BTP chunk orchestration (`_forward_btp`, simulator.py:550-714) with
every compute site on libbtp.so kernels and every boundary on `TPComm` (NCCL on the box):

  attention half  K3 norm1(x) -> K1 down qkv (x rms_loc) -> AR [T,3r]+rider -> K4 fix-up+sigma
                  -> K2 batched up q|k|v -> SDPA -> K1 down o -> AR [T,r] -> K4 sigma
                  -> K2 up o (+x residual in the epilogue) = x_mid
  mlp half        K3 norm2(x_mid) -> K1 down gate|up -> AR [T,2r]+rider -> K4 -> K2 batched up
                  gate|up -> K5 swiglu -> K1 down -> AR [T,r] -> K4 -> K2 up down (+x_mid) = y

Backward mirrors it (the reference has none): each up-projection's input gradient is the
only collective ([T,k*r] all-reduce), sigma-bwd and the online-norm backward are rank-local
(dP = dz/s, dss = -<dz,z>/(2 s^2 d), dx = dh*gamma + 2 x dss), and every weight gradient is
a local split-K tcgen05 GEMM in fp32. The down-factor gradient uses dB_i = (dP^T x_i) * gamma_i
(column scale), so the normalised activations never need to be kept.

Low-rank activation checkpointing (plan.lowrank_ckpt, reference simulator.py:720-921): the
forward keeps only x, the seven rank-r z's and the per-row global RMS; backward recomputes
sigma, the up-projections, attention and swiglu with ZERO collectives.

Layouts (per rank, dl = d/tp, fl = d_ff/tp): activations row-major bf16 [T, width]; the
grouped down weight [k*r, dl] (K-major, so the forward GEMM reads it directly and dgrad reads
it MN-major); up weights [d_out/tp, r]; all weight grads fp32.
"""

from __future__ import annotations

import dataclasses
import functools
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from . import peer
from .attention import Attention
from .comm import TPComm
from .model import DecoderBlockWeights, Variant
from .plan import NormMode, PlanError, ShardPlan, Strategy

BF16 = torch.bfloat16
F32 = torch.float32
# sigma kernel variant per model variant: lax applies no activation (its merge with the previous
# layer's bundle is a plain add after the reduction, simulator.py:260-265)
_VAR = {Variant.SVD: 0, Variant.COLA: 1, Variant.LAX: 0}
# bf16: the training path (tcgen05 GEMMs, bf16 activations, fp32 statistics / accumulation);
# fp32: the parity mode (exact-fp32 SIMT GEMM + fp32 row kernels; north_star 1e-4 tolerance)
PRECISIONS = {"bf16": BF16, "fp32": F32}
# TP = 1: sigma in the down-GEMM epilogue instead of a separate fix-up launch (A/B switch for benches)
FUSE_SIGMA = True
# live collectives: forward chunk boundaries pipelined over this many token slices, so the
# all-reduce of slice c overlaps the down GEMM of slice c+1 (and the fix-up of slice c the
# all-reduce of slice c+1) — the north_star's "overlapped with the adjacent GEMM tiles"
FWD_AR_SLICES = 4
FWD_SLICE_MIN_ROWS = 1024  # below this the launch count outweighs the overlap


_NVTX = os.environ.get("BTP_NVTX", "0") == "1"


def _nvtx(fn):
    """NVTX range around an executor stage (BTP_NVTX=1; e.g. for Nsight Systems timelines): the
    range is named after the stage and the chunk it works on (`names` argument)."""
    if not _NVTX:
        return fn

    @functools.wraps(fn)
    def wrapped(self, *args, **kwargs):
        names = args[0] if args and isinstance(args[0], tuple) else ()
        torch.cuda.nvtx.range_push(f"{fn.__name__.strip('_')}:{'|'.join(names)}:{self.comm.pass_tag}")
        try:
            return fn(self, *args, **kwargs)
        finally:
            torch.cuda.nvtx.range_pop()

    return wrapped


def _pick_splits(tiles: int, k_blocks: int, units: int) -> int:
    """Split-K factor for a weight-gradient GEMM (the reduction runs over the T tokens).

    tiles: 256 x 256 CTA-pair output tiles of one split; units: CTA pairs (SMs / 2). Cost model,
    fitted to measured B200 sweeps (scripts/microbench/gpu_gemm_ab.py, scripts/microbench/gpu_gemm_ab2.py): a launch takes
    waves x (k-blocks per split + ~5 k-blocks of per-tile epilogue / pipeline fill), with
    waves = ceil(tiles * splits / units). Keeps >= 4 k-blocks (256 tokens) per split; ties go to
    fewer splits (less reduce-add traffic)."""
    best, best_cost = 1, None
    for s in range(1, 17):
        kb = -(-k_blocks // s)
        if s > 1 and kb < 4:
            break
        cost = -(-tiles * s // units) * (kb + 5)
        if best_cost is None or cost < best_cost:
            best, best_cost = s, cost
    return best


_BEHIND_TILE_OVERHEAD = 5  # k-block equivalents of per-tile epilogue / pipeline fill in the merged model


def _pick_splits_behind(ahead_kb: list, w_tiles: int, k_blocks: int, units: int) -> int:
    """Split-K factor for weight-gradient tiles launched BEHIND other tiles in the same persistent
    launch (ahead_kb: k-blocks of each tile ahead, in launch order). Tiles go round-robin to the CTA
    pairs; the launch takes the busiest pair's sum of (k-blocks + ~5) per tile (the _pick_splits
    model, with heterogeneous tiles)."""
    best, best_cost = 1, None
    for s in range(1, 17):
        kb = -(-k_blocks // s)
        if s > 1 and kb < 4:
            break
        loads = [0] * units
        for j, c in enumerate(list(ahead_kb) + [kb] * (w_tiles * s)):
            loads[j % units] += c + _BEHIND_TILE_OVERHEAD
        cost = max(loads)
        if best_cost is None or cost < best_cost:
            best, best_cost = s, cost
    return best


@dataclass
class StepStats:
    gemm_launches: int = 0
    kernel_launches: int = 0
    gemm_flops: int = 0


class ExecutorBase:
    """Buffers, GEMM dispatch (+ optional per-launch timing), split-K weight gradients and the
    loss, shared by the BTP executor and the naive-TP / full-rank baselines (baselines.py)."""

    residual_sharded = True
    gemm_timer: list | None = None  # bench instrumentation: (start_event, end_event, flops) per launch
    gemm_log: list | None = None    # bench instrumentation: (problems, flops) of every launch, in order
    fuse_swiglu_bwd = False         # SwiGLU backward in the dgrad GEMM epilogue (False: separate kernel)

    def _setup(self, pl: ShardPlan, comm: TPComm | None, device, eps: float, precision: str = "bf16"):
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        self.precision = precision
        self.act = PRECISIONS[precision]  # activation / GEMM-operand dtype
        self.pl, self.cfg, self.shape = pl, pl.cfg, pl.shape
        self.comm = comm if comm is not None else TPComm(1, 0)
        if self.comm.tp != pl.shape.tp:
            raise PlanError(f"communicator size {self.comm.tp} != plan tp {pl.shape.tp}")
        self.dev = torch.device(device)
        self.eps = eps
        self.tp, self.rank = pl.shape.tp, self.comm.rank
        self.T = pl.shape.tokens
        self.sms = K.num_sms()
        self.stats = StepStats()
        self._buf: dict[str, torch.Tensor] = {}
        self._scratch: dict[str, torch.Tensor] = self._buf   # see share_scratch
        self.saved: dict = {}

    def _dev(self, a, dtype=None) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev, dtype or self.act)

    # ------------------------------------------------------------------ flat parameters + AdamW
    def _flatten_params(self) -> None:
        """Re-home every working weight as a view of ONE flat buffer (GEMM operand dtype) and every
        weight gradient as a view of ONE flat fp32 buffer (segments 8-element aligned), and the
        two gammas likewise, so the optimizer update is a single fused launch per group."""

        def flat(groups, wdtype):
            segs, total = [], 0
            for key, idx, t in groups:
                segs.append((key, idx, t, total))
                total += -(-t.numel() // 8) * 8
            wf = torch.zeros(total, dtype=wdtype, device=self.dev)
            gf = torch.zeros(total, dtype=F32, device=self.dev)
            views = []
            for key, idx, t, off in segs:
                wv = wf[off:off + t.numel()].view(t.shape)
                wv.copy_(t)
                views.append((key, idx, wv, gf[off:off + t.numel()].view(t.shape)))
            return wf, gf, views

        lin = []
        for k, v in self.W.items():
            for i, t in enumerate(v if isinstance(v, list) else [v]):
                lin.append((k, i if isinstance(v, list) else None, t))
        self.w_flat, self.g_flat, views = flat(lin, self.act)
        W, G = {}, {}
        for key, idx, wv, gv in views:
            if idx is None:
                W[key], G[key] = wv, gv
            else:
                W.setdefault(key, []).append(wv)
                G.setdefault(key, []).append(gv)
        self.gam_flat, self.gam_grad_flat, gviews = flat([("gamma1", None, self.gamma1),
                                                          ("gamma2", None, self.gamma2)], F32)
        self.gamma1, self.gamma2 = gviews[0][2], gviews[1][2]
        G["gamma1"], G["gamma2"] = gviews[0][3], gviews[1][3]
        self.W, self.grad = W, G
        self.opt = None

    def optimizer_step(self, lr: float = 1e-4, b1: float = 0.9, b2: float = 0.95, eps: float = 1e-8,
                       wd: float = 0.1) -> None:
        """AdamW on this rank's shard of the parameters (fp32 master + moments, created lazily):
        one fused launch for the linear factors, one for the norm gains (no weight decay)."""
        if self.opt is None:
            z = lambda t: torch.zeros(t.numel(), dtype=F32, device=self.dev)  # noqa: E731
            self.opt = {"master": self.w_flat.float().clone(), "m": z(self.w_flat), "v": z(self.w_flat),
                        "gm": z(self.gam_flat), "gv": z(self.gam_flat),
                        "step": torch.ones(1, dtype=torch.int32, device=self.dev)}  # device counter, 1-based
        self._join_side()
        o = self.opt
        K.adamw(o["master"], o["m"], o["v"], self.g_flat, self.w_flat, lr=lr, step_dev=o["step"], b1=b1, b2=b2,
                eps=eps, wd=wd)
        K.adamw(self.gam_flat, o["gm"], o["gv"], self.gam_grad_flat, self.gam_flat, lr=lr, step_dev=o["step"], b1=b1,
                b2=b2, eps=eps, wd=0.0)
        K.counter_add(o["step"], 1)
        self.stats.kernel_launches += 3

    # ------------------------------------------------------------------ buffers
    def share_scratch(self, scratch: dict) -> None:
        """Home this executor's non-persistent buffers in `scratch`, one dict shared by all blocks
        of a model: forward temporaries (n1, n2, ...), backward scratch and — under low-rank
        checkpointing — every activation the backward recomputes. Only `_persistent` names (what
        the backward reads from the forward, and the block output) stay per block, so an L-block
        model holds L x (persistent set) + ONE scratch set in HBM."""
        self._scratch = scratch

    def _persistent(self, name: str) -> bool:
        return True

    def _store(self, name: str) -> dict:
        if self._scratch is self._buf or self._persistent(name):
            return self._buf
        return self._scratch

    def buf(self, name: str, shape, dtype=None) -> torch.Tensor:
        dtype = dtype or self.act
        pc = getattr(self, "peer", None)
        if pc is not None and pc.has(name):  # symmetric (peer-mapped) buffer of the fused boundaries
            t = pc.buf(name)
            if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
                raise PlanError(f"symmetric buffer {name}: {t.dtype} {tuple(t.shape)} != {dtype} {tuple(shape)}")
            return t
        store = self._store(name)
        t = store.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.empty(shape, device=self.dev, dtype=dtype)
            store[name] = t
        return t

    def _wgrad_parts(self, n_elems: int) -> torch.Tensor:
        t = self._scratch.get("_wg_parts")
        if t is None or t.numel() < n_elems:
            t = torch.empty(n_elems, device=self.dev, dtype=F32)
            self._scratch["_wg_parts"] = t
        return t

    # ------------------------------------------------------------------ GEMM helpers
    def _gemm(self, *probs: K.Gemm) -> None:
        flops = 0
        shapes = []
        for p in probs:
            M = p.a.shape[1] if p.a_mn else p.a.shape[0]
            Kd = p.a.shape[0] if p.a_mn else p.a.shape[1]
            N = p.b.shape[1] if p.b_mn else p.b.shape[0]
            flops += 2 * M * N * Kd
            shapes.append((M, N, Kd, int(p.a_mn), int(p.b_mn), p.splits))
        if self.gemm_log is not None:
            self.gemm_log.append((probs, flops))
        if self.gemm_timer is not None:
            # external=True: inside a CUDA-graph capture these become event-record nodes, so the
            # timings are pure device time (no host launch gaps)
            e0 = torch.cuda.Event(enable_timing=True, external=True)
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            e0.record()
            K.gemm(*probs)
            e1.record()
            self.gemm_timer.append((e0, e1, flops, shapes))
        else:
            K.gemm(*probs)
        self.stats.gemm_launches += 1
        self.stats.kernel_launches += 1
        self.stats.gemm_flops += flops

    # Optionally the weight-gradient GEMMs run on a side stream, concurrently with the main stream's
    # dgrad GEMMs and row kernels: nothing on the main stream consumes a weight gradient before the
    # optimizer, every wgrad input is written once per step, and the side stream is joined at the
    # end of backward (_join_side). Measured on the CoLA-1B TP=1 step it is neutral (4.77 vs
    # 4.77-4.83 ms: the persistent GEMMs already fill the SMs and the 1 kW power cap binds), so
    # it is off by default (`bench.py --concurrent-wgrad` to A/B).
    concurrent_wgrad = False

    def _side(self) -> torch.cuda.Stream:
        s = getattr(self, "_side_stream", None)
        if s is None:
            s = self._side_stream = torch.cuda.Stream(device=self.dev)
        return s

    def _join_side(self) -> None:
        if getattr(self, "_side_pending", False):
            torch.cuda.current_stream(self.dev).wait_stream(self._side_stream)
            self._side_pending = False

    def _gemm_scatter(self, *probs: K.Gemm, owner_buf: str, col0) -> None:
        """A GEMM launch whose epilogue reduce-adds each row block into the owning rank's
        `owner_buf` (peer memory) — the row-parallel partial and its reduce-scatter in one kernel."""
        pc = self.peer
        W = pc.buf(owner_buf).shape[1]
        flops = 0
        for p in probs:
            M = p.a.shape[1] if p.a_mn else p.a.shape[0]
            Kd = p.a.shape[0] if p.a_mn else p.a.shape[1]
            N = p.b.shape[1] if p.b_mn else p.b.shape[0]
            flops += 2 * M * N * Kd
        K.gemm_scatter(*probs, owners=pc.host_ptrs(owner_buf), rows_per_owner=self.T // self.tp, width=W, ld=W,
                       col0=col0)
        self.stats.gemm_launches += 1
        self.stats.kernel_launches += 1
        self.stats.gemm_flops += flops

    def _wgrad(self, pairs, col_scale=None):
        if not self.concurrent_wgrad:
            return self._wgrad_now(pairs, col_scale)
        side = self._side()
        side.wait_stream(torch.cuda.current_stream(self.dev))  # inputs produced so far on the main stream
        with torch.cuda.stream(side):
            self._wgrad_now(pairs, col_scale)
        self._side_pending = True

    # With no collective to start between them and no side stream, a dgrad and its chunk's
    # independent weight gradient(s) go out as ONE grouped launch (<= 8 problems): the weight-gradient
    # split tiles fill the dgrad's last wave and one launch's prologue / pipeline fill / drain is
    # saved. (_up_bwd merges only without live collectives: there the boundary all-reduce of the
    # dgrad output starts before the weight gradient and overlaps it.) `merge_bwd_gemms = False`
    # restores two launches (A/B).
    merge_bwd_gemms = True

    def _dgrad_wgrad(self, dgrad_probs, pairs, col_scale=None):
        """dgrad problem(s) then the weight gradient(s) of `pairs` (see _wgrad_now), merged into one
        launch when nothing needs the dgrad output early."""
        cap = 4 if dgrad_probs[0].a.dtype == F32 else 8  # problems per launch: fp32 SIMT GEMM / tcgen05 GEMM
        if not self.merge_bwd_gemms or self.concurrent_wgrad or len(dgrad_probs) + len(pairs) > cap:
            self._gemm(*dgrad_probs)
            self._wgrad(pairs, col_scale)
            return
        units = max(self.sms // 2, 1)
        ahead = []
        for p in dgrad_probs:
            M = p.a.shape[1] if p.a_mn else p.a.shape[0]
            Kd = p.a.shape[0] if p.a_mn else p.a.shape[1]
            N = p.b.shape[1] if p.b_mn else p.b.shape[0]
            ahead += [(Kd + 63) // 64] * (math.ceil(M / 256) * math.ceil(N / 256))
        T = pairs[0][0].shape[0]
        w_tiles = sum(math.ceil(dy.shape[1] / 256) * math.ceil(x.shape[1] / 256) for dy, x, _ in pairs)
        splits = _pick_splits_behind(ahead, w_tiles, (T + 63) // 64, units)
        if splits > 1:
            for _, _, o in pairs:
                K.zero(o)
        self._gemm(*dgrad_probs, *[K.Gemm(dy, x, o, a_mn=True, b_mn=True, splits=splits, col_scale=col_scale)
                                   for dy, x, o in pairs])

    def _wgrad_now(self, pairs, col_scale=None):
        """pairs: list of (dY [T, M] (MN-major A), X [T, N] (MN-major B), out fp32 [M, N]).
        out = (dY^T X) (* col_scale). With split-K every split TMA-reduce-adds its fp32 tile into the
        zeroed gradient in L2; the order of those adds across CTAs is not fixed, so split weight
        gradients are reproducible to fp32 rounding, not bitwise, from run to run."""
        T = pairs[0][0].shape[0]
        kb = (T + 63) // 64
        tiles = sum(math.ceil(dy.shape[1] / 256) * math.ceil(x.shape[1] / 256) for dy, x, _ in pairs)
        splits = _pick_splits(tiles, kb, max(self.sms // 2, 1))
        if splits == 1:
            self._gemm(*[K.Gemm(dy, x, o, a_mn=True, b_mn=True, col_scale=col_scale) for dy, x, o in pairs])
            return
        # split-K: every split adds its fp32 tile into the zeroed gradient with the TMA reduce-add
        for _, _, o in pairs:
            K.zero(o)
        self._gemm(*[K.Gemm(dy, x, o, a_mn=True, b_mn=True, splits=splits, col_scale=col_scale)
                     for dy, x, o in pairs])

    # ------------------------------------------------------------------ loss / accounting
    def loss_device(self, y: torch.Tensor, G: torch.Tensor) -> torch.Tensor:
        """L = sum(y * G) over the logical [T, d] (builder-defined; the reference has no loss).
        Device dot product + deterministic reduction into a 1-element fp32 buffer (no sync)."""
        part = self.buf("loss_parts", (4 * self.sms,), F32)
        nb = K.dot(y, G, part)
        out = self.buf("loss", (1,), F32)
        K.reduce_rows(part[:nb].view(nb, 1, 1), out.view(1, 1))
        self.stats.kernel_launches += 2
        if self.comm.live and self.residual_sharded:
            import torch.distributed as dist

            dist.all_reduce(out, group=self.comm.group)  # loss over the TP group's d-shards (not logged)
        return out

    def loss(self, y: torch.Tensor, G: torch.Tensor) -> float:
        return float(self.loss_device(y, G).item())

    def saved_activation_elements(self) -> int:
        """Elements of activations held between forward and backward (distinct storages)."""
        seen, total = set(), 0
        for v in self.saved.values():
            ts = v if isinstance(v, (list, tuple)) else [v]
            for t in ts:
                if isinstance(t, torch.Tensor):
                    key = t.untyped_storage().data_ptr()
                    if key not in seen:
                        seen.add(key)
                        total += t.untyped_storage().nbytes() // t.element_size()
        return total

    def saved_activation_bytes(self) -> int:
        """Bytes of activations held between forward and backward (distinct storages)."""
        seen, total = set(), 0
        for v in self.saved.values():
            ts = v if isinstance(v, (list, tuple)) else [v]
            for t in ts:
                if isinstance(t, torch.Tensor):
                    key = t.untyped_storage().data_ptr()
                    if key not in seen:
                        seen.add(key)
                        total += t.untyped_storage().nbytes()
        return total


class BTPBlockExecutor(ExecutorBase):
    """One rank's shard of a low-rank (svd/cola/lax) block under a BTP plan."""

    # "fp32": the forward chunk boundaries (NCCL path, tp > 1) reduce an fp32 partial — the down
    # GEMM writes P in fp32 and btp_fixup_sigma_f32in rounds the cross-rank sum to bf16 once —
    # instead of a bf16 all-reduce that rounds at every ring hop (2x the forward boundary bytes).
    # Measured (scripts/margin_probe2.py): the worst TP=8 parity error drops 1.86e-2 -> 1.58e-2 at
    # CoLA-7B widths and 1.98e-2 -> 1.78e-2 at CoLA-60M; an fp32 BACKWARD reduction does not move it.
    boundary_dtype = "bf16"

    def __init__(self, pl: ShardPlan, block: DecoderBlockWeights, comm: TPComm | None = None,
                 device: torch.device | str = "cuda", eps: float = 1e-6, attn_backend: str = "auto",
                 precision: str = "bf16"):
        if pl.strategy is not Strategy.BOTTLENECK:
            raise PlanError(f"BTPBlockExecutor needs a btp plan, got {pl.strategy.value}")
        if block.variant is not pl.variant:
            raise PlanError(f"plan variant {pl.variant.value} != block variant {block.variant.value}")
        if pl.variant not in _VAR:
            raise PlanError(f"variant {pl.variant.value} is not supported on the device path (svd, cola, lax)")
        self._setup(pl, comm, device, eps, precision)
        self.var = _VAR[pl.variant]
        # lax (simulator.py:247-265): a = z + h_prev[name] after the reduction, h_cur = z. The
        # bundle is replicated like z; set_h_prev() stages it per chunk ([T, k*r] like P).
        self.lax = pl.variant is Variant.LAX
        self.has_h_prev = False
        self.h_prev: dict | None = None
        self.dh_prev: dict | None = None
        self.dh_cur_in: dict | None = None  # lax models: dL/dh_cur from the next layer's merge
        self.online = pl.norm_mode is NormMode.ONLINE
        self.grouping = pl.grouping
        self.ckpt = pl.lowrank_ckpt
        cfg, tp = self.cfg, self.tp
        self.r, self.d, self.d_ff = cfg.r, cfg.d, cfg.d_ff
        self.dl, self.fl, self.hl = cfg.d // tp, cfg.d_ff // tp, cfg.heads // tp
        # d_ff shard padded to a multiple of 8 (16-byte TMA row strides; e.g. CoLA-1B at TP=8 has
        # fl = 684): zero rows in the gate/up up-factors and zero columns in the down down-factor
        # make the padding exact (g = u = act = 0 there, and their gradients are 0).
        self.flp = -(-self.fl // 8) * 8
        self.attn = Attention(pl.shape.b, pl.shape.s, self.hl, cfg.head_dim,
                              "fp32" if precision == "fp32" else attn_backend)
        self.attn.stats = self.stats
        # sigma in the down-GEMM epilogue (GEMM kernel epilogue 1): TP = 1 only (at TP > 1 the
        # all-reduce sits between GEMM and sigma), cola, bf16, crossgate halves in 64-column blocks
        self.fuse_sigma = (FUSE_SIGMA and precision == "bf16" and tp == 1 and self.var == 1 and self.r % 128 == 0
                           and not self.comm.live)
        # token slices of the pipelined forward boundaries (live collectives only; 128-row multiples)
        self.fwd_slices = 1
        if self.comm.live and self.grouping:
            for c in (FWD_AR_SLICES, 2):
                if c > 1 and self.T % (c * 128) == 0 and self.T // c >= FWD_SLICE_MIN_ROWS:
                    self.fwd_slices = c
                    break
        # chunk boundaries over peer memory (csrc/peer.cu): one fused reduce-scatter -> fix-up/sigma
        # -> all-gather kernel per boundary and pass instead of an NCCL all-reduce + fix-up launch
        self.peer = getattr(self.comm, "peer", None)
        if self.peer is not None:
            if not (self.grouping and self.online and not self.ckpt and precision == "bf16"):
                raise PlanError("peer-memory boundaries need grouping, the online norm, bf16 and no low-rank ckpt")
            if self.T % tp:
                raise PlanError(f"peer-memory boundaries need T={self.T} divisible by tp={tp}")
            self.fuse_sigma = False
            self.peer.setup(self._peer_specs())
        self._load_weights(block)

    CHUNKS = (("q", "k", "v"), ("o",), ("gate", "up"), ("down",))

    # per-block buffers when blocks share scratch (share_scratch): the block output, the norm
    # statistics, the stored z's (= the forward all-reduce buffers), the lax bundle and its
    # gradient; without low-rank ckpt also every activation the backward reads
    _KEEP = frozenset({"y", "s1", "s2", "rl1", "rl2"})
    _KEEP_PREFIX = ("P_", "P3_", "zown_", "hp_", "dPlax_")
    _KEEP_NO_CKPT = frozenset({"qkv", "attn", "x_mid", "gu", "act"})
    _KEEP_NO_CKPT_PREFIX = ("a_", "alax_")

    def _persistent(self, name: str) -> bool:
        if name in self._KEEP or name.startswith(self._KEEP_PREFIX):
            return True
        # lax: dL/dh_prev are views of the reduced dA, read by the PREVIOUS block's backward
        # (its dL/dh_cur) after this block's backward returned — they must outlive the scratch
        if self.lax and name.startswith(("dA_", "dA3_")):
            return True
        if self.ckpt:
            return False
        return name in self._KEEP_NO_CKPT or name.startswith(self._KEEP_NO_CKPT_PREFIX)

    def _peer_specs(self):
        """Symmetric buffers of the peer boundaries, identical (names, shapes, order) on every rank:
        per chunk the down-GEMM partial P, the pushed activation a, the up-GEMM dgrad partial dA and
        the pushed dP; the online-norm riders ss1/ss2 and the pushed norm-statistic grads dss1/dss2."""
        T, r, specs = self.T, self.r, []
        scatter = getattr(self.comm.peer, "scatter", False)
        for names in self.CHUNKS:
            key, W = "_".join(names), len(names) * self.r
            if scatter:  # reduce targets: this rank's owned rows, written by every rank's scatter GEMM
                specs += [(f"R_{key}", (T // self.tp, W), F32), (f"RdA_{key}", (T // self.tp, W), F32)]
                specs += [(f"{pre}_{key}", (T, W), self.act) for pre in ("a", "dP")]
            else:
                specs += [(f"{pre}_{key}", (T, W), self.act) for pre in ("P", "a", "dA", "dP")]
        specs += [(nm, (T,), F32) for nm in ("ss1", "ss2", "dss1", "dss2")]
        return specs

    # ------------------------------------------------------------------ weights
    def _load_weights(self, block: DecoderBlockWeights) -> None:
        sl = slice(self.rank * self.dl, (self.rank + 1) * self.dl)
        fsl = slice(self.rank * self.fl, (self.rank + 1) * self.fl)
        B = {n: t.values for n, t in block.down_factors.items()}
        A = {n: t.values for n, t in block.up_factors.items()}

        def dev(a, dtype=None):
            return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev, dtype or self.act)

        pad = self.flp - self.fl

        def pad_rows(a):  # [fl, r] -> [flp, r]
            return np.pad(a, ((0, pad), (0, 0))) if pad else a

        def pad_cols(a):  # [r, fl] -> [r, flp]
            return np.pad(a, ((0, 0), (0, pad))) if pad else a

        self.W = {
            "d_qkv": dev(np.concatenate([B[n][:, sl] for n in ("q", "k", "v")], axis=0)),   # [3r, dl]
            "u_qkv": dev(np.stack([A[n][sl, :] for n in ("q", "k", "v")])),                 # [3, dl, r]
            "d_o": dev(B["o"][:, sl]),                                                       # [r, dl]
            "u_o": dev(A["o"][sl, :]),                                                       # [dl, r]
            "d_gu": dev(np.concatenate([B[n][:, sl] for n in ("gate", "up")], axis=0)),     # [2r, dl]
            "u_gu": dev(np.stack([pad_rows(A[n][fsl, :]) for n in ("gate", "up")])),        # [2, flp, r]
            "d_d": dev(pad_cols(B["down"][:, fsl])),                                         # [r, flp]
            "u_d": dev(A["down"][sl, :]),                                                    # [dl, r]
        }
        self.gamma1 = dev(block.gamma1.values[sl], F32)
        self.gamma2 = dev(block.gamma2.values[sl], F32)
        self.grad = {k: torch.zeros(v.shape, device=self.dev, dtype=F32) for k, v in self.W.items()}
        self.grad["gamma1"] = torch.zeros(self.dl, device=self.dev, dtype=F32)
        self.grad["gamma2"] = torch.zeros(self.dl, device=self.dev, dtype=F32)
        self._flatten_params()

    def weight_grads_by_name(self) -> dict[str, dict[str, np.ndarray]]:
        """Rank-local gradients keyed like the reference block: {'A': {name: [d_out/tp, r]},
        'B': {name: [r, d_in/tp]}, 'gamma1': [dl], 'gamma2': [dl]} (float64 host copies)."""
        g = {k: v.double().cpu().numpy() for k, v in self.grad.items()}
        r = self.r
        out = {"A": {}, "B": {}, "gamma1": g["gamma1"], "gamma2": g["gamma2"]}
        for i, n in enumerate(("q", "k", "v")):
            out["B"][n] = g["d_qkv"][i * r:(i + 1) * r]
            out["A"][n] = g["u_qkv"][i]
        for i, n in enumerate(("gate", "up")):
            out["B"][n] = g["d_gu"][i * r:(i + 1) * r]
            out["A"][n] = g["u_gu"][i][:self.fl]
        out["B"]["o"], out["A"]["o"] = g["d_o"], g["u_o"]
        out["B"]["down"], out["A"]["down"] = g["d_d"][:, :self.fl], g["u_d"]
        return out

    # ------------------------------------------------------------------ forward pieces
    @_nvtx
    def _norm(self, x, gamma, tag):
        """Online: n = x*gamma/rms_loc, ss -> rider. Sync: stat AR then global normalisation."""
        T, dl = self.T, self.dl
        n = self.buf(f"n{tag}", (T, dl))
        ss = self.buf(f"ss{tag}", (T,), F32)
        if self.online:
            rl = self.buf(f"rl{tag}", (T,), F32)
            K.rmsnorm_residual(x, gamma, n_out=n, ss_out=ss, rl_out=rl, eps=self.eps)
            self.stats.kernel_launches += 1
            return n, ss, rl, None
        K.rmsnorm_residual(x, gamma, ss_out=ss, eps=self.eps)
        self.comm.all_reduce(ss, f"norm{tag}-stat", tag="block")
        s = self.buf(f"s{tag}", (T,), F32)
        K.rmsnorm_apply(x, gamma, ss, self.d, n, rms_out=s, eps=self.eps)
        self.stats.kernel_launches += 2
        return n, ss, None, s

    @_nvtx
    def _down_boundary(self, names, n_in, W, ss, rl, s_tag, norm_chunk: bool):
        """Row-parallel down GEMM(s) -> all-reduce(s) -> fix-up + sigma.
        Returns (z views, a views, P storage); z aliases the all-reduce buffer."""
        T, r, k = self.T, self.r, len(names)
        row_scale = rl if (norm_chunk and self.online) else None
        ss_total = ss if (norm_chunk and self.online) else None
        s_out = self.buf(f"s{s_tag}", (T,), F32) if (norm_chunk and self.online) else None
        if self.peer is not None:
            return self._down_boundary_peer(names, n_in, W, rl, s_tag, norm_chunk)
        a_store = self.buf(f"a_{'_'.join(names)}", (T, k * r)) if self.var == 1 else None
        if self.fuse_sigma:
            return self._down_boundary_fused(names, n_in, W, ss, rl, s_tag, norm_chunk, a_store)
        if self.fwd_slices > 1:
            return self._down_boundary_sliced(names, n_in, W, ss, rl, s_out, norm_chunk, a_store)
        f32 = self.boundary_dtype == "fp32" and self.comm.live
        if self.grouping or k == 1:
            P = self.buf(f"P_{'_'.join(names)}", (T, k * r))
            Pr = self.buf(f"Pf_{'_'.join(names)}", (T, k * r), F32) if f32 else P  # the reduced buffer
            self._gemm(K.Gemm(n_in, W, Pr, row_scale=row_scale))
            if ss_total is not None:
                self.comm.all_reduce_coalesced(Pr, ss, names[0] if k == 1 else self._gid(names))
            else:
                self.comm.all_reduce(Pr, names[0] if k == 1 else self._gid(names))
            if self.var == 1 or ss_total is not None or f32:
                K.fixup_sigma(Pr, r=r, nproj=k, variant=self.var, z_out=P, a_out=a_store, ss_total=ss_total,
                              d=self.d, s_out=s_out, eps=self.eps)
                self.stats.kernel_launches += 1
            z = [P[:, i * r:(i + 1) * r] for i in range(k)]
            a = [a_store[:, i * r:(i + 1) * r] for i in range(k)] if a_store is not None else z
            return z, a, P
        # ungrouped: one GEMM + one collective per projection (reference simulator.py:623-639)
        P3 = self.buf(f"P3_{'_'.join(names)}", (k, T, r))
        Pr3 = self.buf(f"Pf3_{'_'.join(names)}", (k, T, r), F32) if f32 else P3
        z, a = [], []
        for i, nm in enumerate(names):
            self._gemm(K.Gemm(n_in, W[i * r:(i + 1) * r], Pr3[i], row_scale=row_scale))
            if ss_total is not None and i == 0:
                self.comm.all_reduce_coalesced(Pr3[i], ss, nm)
            else:
                self.comm.all_reduce(Pr3[i], nm)
            if self.var == 1 or ss_total is not None or f32:
                a_i = a_store[:, i * r:(i + 1) * r] if a_store is not None else None
                K.fixup_sigma(Pr3[i], r=r, nproj=1, variant=self.var, z_out=P3[i], a_out=a_i, ss_total=ss_total,
                              d=self.d, s_out=s_out if i == 0 else None, eps=self.eps)
                self.stats.kernel_launches += 1
            z.append(P3[i])
            a.append(a_store[:, i * r:(i + 1) * r] if a_store is not None else P3[i])
        return z, a, P3

    def _down_boundary_fused(self, names, n_in, W, ss, rl, s_tag, norm_chunk, a_store):
        """TP = 1: no all-reduce separates the down GEMM from sigma, so the GEMM epilogue writes
        z and a = crossgate(z) directly (no P round trip, no fix-up launch). With a single rank,
        rms_loc is the global rms, so z needs no rescale and s = rms_loc. The (no-op) collectives
        are still recorded, in plan order."""
        T, r, k = self.T, self.r, len(names)
        if norm_chunk and self.online:
            self._store(f"s{s_tag}")[f"s{s_tag}"] = rl
        if self.grouping or k == 1:
            P = self.buf(f"P_{'_'.join(names)}", (T, k * r))
            self._gemm(K.Gemm(n_in, W, P, sigma=(a_store, r // 2)))
            gid = names[0] if k == 1 else self._gid(names)
            if norm_chunk and self.online:
                self.comm.all_reduce_coalesced(P, ss, gid)
            else:
                self.comm.all_reduce(P, gid)
            return ([P[:, i * r:(i + 1) * r] for i in range(k)], [a_store[:, i * r:(i + 1) * r] for i in range(k)],
                    P)
        P3 = self.buf(f"P3_{'_'.join(names)}", (k, T, r))
        for i, nm in enumerate(names):
            self._gemm(K.Gemm(n_in, W[i * r:(i + 1) * r], P3[i], sigma=(a_store[:, i * r:(i + 1) * r], r // 2)))
            if norm_chunk and self.online and i == 0:
                self.comm.all_reduce_coalesced(P3[i], ss, nm)
            else:
                self.comm.all_reduce(P3[i], nm)
        return [P3[i] for i in range(k)], [a_store[:, i * r:(i + 1) * r] for i in range(k)], P3

    def _down_boundary_sliced(self, names, n_in, W, ss, rl, s_out, norm_chunk, a_store):
        """Grouped boundary with live collectives, pipelined over token slices: the down GEMM of
        slice c+1 runs while slice c's all-reduce (+ rider) is in flight on NCCL's stream; slice c's
        fix-up + sigma runs once its reduction landed, overlapping slice c+1's. Rows are
        independent, so the result is bit-identical to the unsliced boundary; the collective log
        keeps ONE record per chunk boundary (the logical collective of the reference)."""
        T, r, k, C = self.T, self.r, len(names), self.fwd_slices
        online = norm_chunk and self.online
        f32 = self.boundary_dtype == "fp32"
        P = self.buf(f"P_{'_'.join(names)}", (T, k * r))
        Pr = self.buf(f"Pf_{'_'.join(names)}", (T, k * r), F32) if f32 else P  # the reduced buffer
        gid = names[0] if k == 1 else self._gid(names)
        rows = T // C
        handles = []
        for c in range(C):
            sl = slice(c * rows, (c + 1) * rows)
            self._gemm(K.Gemm(n_in[sl], W, Pr[sl], row_scale=rl[sl] if online else None))
            if online:
                handles.append(self.comm.all_reduce_coalesced_start(Pr[sl], ss[sl], gid, record=False))
            else:
                handles.append(self.comm.all_reduce_start(Pr[sl], gid, record=False))
        if online:
            self.comm.record("all-reduce-coalesced", gid, T * k * r, extras=(("fused-stat", T),))
        else:
            self.comm.record("all-reduce", gid, T * k * r)
        for c in range(C):
            self.comm.wait(handles[c])
            if self.var == 1 or online or f32:
                sl = slice(c * rows, (c + 1) * rows)
                K.fixup_sigma(Pr[sl], r=r, nproj=k, variant=self.var, z_out=P[sl],
                              a_out=a_store[sl] if a_store is not None else None, ss_total=ss[sl] if online else None,
                              d=self.d, s_out=s_out[sl] if s_out is not None else None, eps=self.eps)
                self.stats.kernel_launches += 1
        z = [P[:, i * r:(i + 1) * r] for i in range(k)]
        a = [a_store[:, i * r:(i + 1) * r] for i in range(k)] if a_store is not None else z
        return z, a, P

    def _down_boundary_peer(self, names, n_in, W, rl, s_tag, norm_chunk):
        """Row-parallel down GEMM into the symmetric P, then ONE kernel: pull-reduce this rank's
        T/tp rows of every rank's P (+ the ss rider), z = P/s and a = sigma(z) on them, push a into
        every rank's a. z and s stay for the owned rows only (the backward needs nothing else)."""
        T, r, k, tp = self.T, self.r, len(names), self.tp
        key = "_".join(names)
        pc = self.peer
        z_own = self.buf(f"zown_{key}", (T // tp, k * r))
        s_own = self.buf(f"s{s_tag}", (T // tp,), F32) if norm_chunk else None
        a = self.buf(f"a_{key}", (T, k * r))
        ss_name = f"ss{s_tag}" if norm_chunk else None
        if pc.scatter:
            # ONE kernel for GEMM + reduce-scatter: every output row block is reduce-added into its
            # owner's R buffer over NVLink as the tiles finish; then only owned rows are read
            self._gemm_scatter(K.Gemm(n_in, W, None, row_scale=rl if norm_chunk else None), owner_buf=f"R_{key}",
                               col0=[0])
            pc.exchange(peer.READY)
            peer.boundary_fwd_local(pc, f"R_{key}", ss_name, T, k * r, r, self.var, self.d, self.eps, z_own, s_own,
                                    f"a_{key}")
        else:
            P = self.buf(f"P_{key}", (T, k * r))
            self._gemm(K.Gemm(n_in, W, P, row_scale=rl if norm_chunk else None))
            pc.exchange(peer.READY)
            peer.boundary_fwd(pc, f"P_{key}", ss_name, T, k * r, r, self.var, self.d, self.eps, z_own, s_own,
                              f"a_{key}")
        pc.exchange(peer.DONE)
        self.stats.kernel_launches += 5
        gid = names[0] if k == 1 else self._gid(names)
        if norm_chunk:
            self.comm.trace.emit("all-reduce-coalesced", gid, "block", T * k * r, self.comm.pass_tag,
                                 extras=(("fused-stat", T),))
        else:
            self.comm.trace.emit("all-reduce", gid, "block", T * k * r, self.comm.pass_tag)
        return ([z_own[:, i * r:(i + 1) * r] for i in range(k)], [a[:, i * r:(i + 1) * r] for i in range(k)], z_own)

    @staticmethod
    def _gid(names) -> str:
        return {("q", "k", "v"): "qkv", ("gate", "up"): "gate_up"}[tuple(names)]

    # ------------------------------------------------------------------ lax h bundle
    def set_h_prev(self, h_prev) -> None:
        """Stage the previous layer's lax bundle {projection: [T, r]} (host or device arrays,
        replicated on every rank) for the next forward; None = the first-layer boundary (a = z,
        bitwise the svd block, reference test_model.py:182-192)."""
        if h_prev is None:
            self.set_h_prev_device(None)
            return
        T, r = self.T, self.r
        views = {}
        for names in self.CHUNKS:
            hp = self.buf(f"hp_{'_'.join(names)}", (T, len(names) * r))
            for i, n in enumerate(names):
                v = h_prev[n]
                v = torch.as_tensor(np.asarray(v).reshape(T, r)) if not isinstance(v, torch.Tensor) else v.reshape(T, r)
                hp[:, i * r:(i + 1) * r].copy_(v.to(self.dev, self.act), non_blocking=True)
                views[n] = hp[:, i * r:(i + 1) * r]
        self.set_h_prev_device(views)

    def set_h_prev_device(self, views) -> None:
        """The bundle as device [T, r] views that stay valid through forward AND backward (a
        multi-layer lax model passes the previous block's h_cur views: no copy)."""
        if views is None:
            self.h_prev = None
            self.has_h_prev = False
            return
        if not self.lax:
            raise PlanError(f"h_prev is a lax input; this block is {self.pl.variant.value}")
        if self.peer is not None:
            raise PlanError("lax with an h bundle runs on the NCCL boundaries (the peer kernels push a = z)")
        self.h_prev = dict(views)
        self.has_h_prev = True

    @staticmethod
    def _blocks_of(views, T, r):
        """[T, k*r] tensor whose column blocks are `views`, or None if they are not laid out so."""
        v0, k = views[0], len(views)
        if k == 1:
            return v0
        if v0.stride() != (k * r, 1) or any(v.data_ptr() != v0.data_ptr() + i * r * v0.element_size()
                                             for i, v in enumerate(views)):
            return None
        return v0.as_strided((T, k * r), (k * r, 1))

    def _lax_add(self, a_views, b_views, out_name, names):
        """out[:, i*r:(i+1)*r] = a_i + b_i (btp_add; one launch when both sides are [T, k*r] blocks)."""
        T, r, k = self.T, self.r, len(names)
        out = self.buf(out_name, (T, k * r))
        A, B = self._blocks_of(a_views, T, r), self._blocks_of(b_views, T, r)
        if A is not None and B is not None:
            K.add(A, B, out)
            self.stats.kernel_launches += 1
        else:
            for i in range(k):
                K.add(a_views[i], b_views[i], out[:, i * r:(i + 1) * r])
                self.stats.kernel_launches += 1
        return out

    def _lax_merge(self, names, z_views, out_name):
        """a = z + h_prev per projection into `out_name` [T, k*r]."""
        out = self._lax_add(z_views, [self.h_prev[n] for n in names], out_name, names)
        return [out[:, i * self.r:(i + 1) * self.r] for i in range(len(names))]

    def _a_input(self, names, z_views, a_views):
        """What the up-projection consumes; records the lax h_cur (= z, before the merge)."""
        if not self.lax:
            return a_views
        for n, a in zip(names, a_views):  # a == z for lax (no sigma); full rows in every mode
            self.h_cur[n] = a
        if not self.has_h_prev:
            return a_views
        return self._lax_merge(names, a_views, f"alax_{'_'.join(names)}")

    def _sigma_only(self, z_views, names, out_name):
        """a = sigma(z) for stored z (checkpoint recompute); svd: a = z; lax: z (+ h_prev)."""
        if self.var == 0:
            if self.lax and self.has_h_prev:
                return self._lax_merge(names, z_views, out_name)
            return z_views
        T, r, k = self.T, self.r, len(z_views)
        a_store = self.buf(out_name, (T, k * r))
        for i, z in enumerate(z_views):
            K.fixup_sigma(z, r=r, nproj=1, variant=1, z_out=z, a_out=a_store[:, i * r:(i + 1) * r])
            self.stats.kernel_launches += 1
        return [a_store[:, i * r:(i + 1) * r] for i in range(k)]

    @_nvtx
    def _up(self, a_list, W_list, outs, resid=None):
        probs = [K.Gemm(a, w, o, resid=resid) for a, w, o in zip(a_list, W_list, outs)]
        if self.grouping:
            self._gemm(*probs)
        else:
            for p in probs:
                self._gemm(p)

    # ------------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: this rank's residual shard [T, d/tp] bf16. Returns y shard [T, d/tp] bf16."""
        T, dl, fl, r = self.T, self.dl, self.flp, self.r
        if tuple(x.shape) != (T, dl) or x.dtype != self.act:
            raise PlanError(f"x shard must be {self.act} [{T}, {dl}], got {x.dtype} {tuple(x.shape)}")
        self.comm.pass_tag = "forward"
        W = self.W
        S = {"x": x}
        self.h_cur = {}
        # ---- attention half
        n1, ss1, rl1, s1 = self._norm(x, self.gamma1, 1)
        z_qkv, a_qkv, P_qkv = self._down_boundary(("q", "k", "v"), n1, W["d_qkv"], ss1, rl1, 1, True)
        a_qkv = self._a_input(("q", "k", "v"), z_qkv, a_qkv)
        S["s1"] = s1 if s1 is not None else self._store("s1")["s1"]
        qkv = self.buf("qkv", (3, T, dl))
        self._up(a_qkv, [W["u_qkv"][i] for i in range(3)], [qkv[i] for i in range(3)])
        attn, actx = self.attn.forward(qkv[0], qkv[1], qkv[2])
        self._store("attn")["attn"] = attn
        z_o, a_o, P_o = self._down_boundary(("o",), attn, W["d_o"], None, None, 0, False)
        a_o = self._a_input(("o",), z_o, a_o)
        x_mid = self.buf("x_mid", (T, dl))
        self._up(a_o, [W["u_o"]], [x_mid], resid=x)
        # ---- mlp half
        n2, ss2, rl2, s2 = self._norm(x_mid, self.gamma2, 2)
        z_gu, a_gu, P_gu = self._down_boundary(("gate", "up"), n2, W["d_gu"], ss2, rl2, 2, True)
        a_gu = self._a_input(("gate", "up"), z_gu, a_gu)
        S["s2"] = s2 if s2 is not None else self._store("s2")["s2"]
        gu = self.buf("gu", (2, T, fl))
        self._up(a_gu, [W["u_gu"][0], W["u_gu"][1]], [gu[0], gu[1]])
        act = self.buf("act", (T, fl))
        K.swiglu(gu[0], gu[1], act)
        self.stats.kernel_launches += 1
        z_d, a_d, P_d = self._down_boundary(("down",), act, W["d_d"], None, None, 0, False)
        a_d = self._a_input(("down",), z_d, a_d)
        y = self.buf("y", (T, dl))
        self._up(a_d, [W["u_d"]], [y], resid=x_mid)
        # ---- what backward keeps
        S.update(P_qkv=P_qkv, z_qkv=z_qkv, P_o=P_o, z_o=z_o, P_gu=P_gu, z_gu=z_gu, P_d=P_d, z_d=z_d)
        if not self.ckpt:
            S.update(a_qkv=a_qkv, qkv=qkv, attn=attn, actx=actx, a_o=a_o, x_mid=x_mid, a_gu=a_gu, gu=gu, act=act,
                     a_d=a_d)
        self.saved = S
        return y

    def capture_workspaces(self) -> dict[str, np.ndarray]:
        """This rank's intermediates under the reference's workspace names (simulator.py:561-708),
        as float64 host arrays. `o` and `mlp` are fused into the residual epilogue on the hot path,
        so they are recomputed here by one extra (unfused) GEMM each, for parity checks only."""
        S, T, r = self.saved, self.T, self.r
        names3, names2 = ("q", "k", "v"), ("gate", "up")
        ws = {"x": S["x"]}
        get = lambda n: self._store(n)[n]  # noqa: E731
        ws["n1"], ws["n2"] = get("n1"), get("n2")
        qkv, gu = get("qkv"), get("gu")
        for i, n in enumerate(names3):
            ws[n] = qkv[i]
        ws["gate"], ws["up"] = gu[0][:, :self.fl], gu[1][:, :self.fl]
        ws["attn"] = S.get("attn", self._store("attn").get("attn"))
        ws["x_mid"], ws["act"], ws["y"] = get("x_mid"), get("act")[:, :self.fl], get("y")
        zs = {n: S["z_qkv"][i] for i, n in enumerate(names3)}
        zs.update({n: S["z_gu"][i] for i, n in enumerate(names2)})
        zs["o"], zs["down"] = S["z_o"][0], S["z_d"][0]
        for n, z in zs.items():
            ws[f"z_{n}"] = z
        if self.var == 1 or (self.lax and self.has_h_prev):
            pre = "a_" if self.var == 1 else "alax_"
            for key, names in ((pre + "q_k_v", names3), (pre + "gate_up", names2), (pre + "o", ("o",)),
                               (pre + "down", ("down",))):
                a = get(key)
                for i, n in enumerate(names):
                    ws[f"a_in_{n}"] = a[:, i * r:(i + 1) * r]
        if not self.online:
            ws["norm1-rms"], ws["norm2-rms"] = S["s1"].view(T, 1), S["s2"].view(T, 1)
        a_o = ws.get("a_in_o", zs["o"])
        a_d = ws.get("a_in_down", zs["down"])
        o = torch.empty(T, self.dl, device=self.dev, dtype=self.act)
        mlp = torch.empty(T, self.dl, device=self.dev, dtype=self.act)
        K.gemm(K.Gemm(a_o, self.W["u_o"], o))
        K.gemm(K.Gemm(a_d, self.W["u_d"], mlp))
        ws["o"], ws["mlp"] = o, mlp
        torch.cuda.synchronize(self.dev)
        return {k: v.double().cpu().numpy() for k, v in ws.items() if v is not None}

    # ------------------------------------------------------------------ recompute (ckpt)
    def _recompute_mlp_inputs(self):
        """Rebuild x_mid, a_gu, gate/up, act, a_d from x and the stored z's; no collective."""
        S, W, T, dl, fl = self.saved, self.W, self.T, self.dl, self.flp
        self.comm.pass_tag = "reforward"
        a_o = self._sigma_only(S["z_o"], ("o",), "a_o_rc")
        x_mid = self.buf("x_mid", (T, dl))
        self._up(a_o, [W["u_o"]], [x_mid], resid=S["x"])
        a_gu = self._sigma_only(S["z_gu"], ("gate", "up"), "a_gu_rc")
        gu = self.buf("gu", (2, T, fl))
        self._up(a_gu, [W["u_gu"][0], W["u_gu"][1]], [gu[0], gu[1]])
        act = self.buf("act", (T, fl))
        K.swiglu(gu[0], gu[1], act)
        self.stats.kernel_launches += 1
        a_d = self._sigma_only(S["z_d"], ("down",), "a_d_rc")
        S.update(a_o=a_o, x_mid=x_mid, a_gu=a_gu, gu=gu, act=act, a_d=a_d)

    def _recompute_attn_inputs(self):
        S, W, T, dl = self.saved, self.W, self.T, self.dl
        self.comm.pass_tag = "reforward"
        a_qkv = self._sigma_only(S["z_qkv"], ("q", "k", "v"), "a_qkv_rc")
        qkv = self.buf("qkv", (3, T, dl))
        self._up(a_qkv, [W["u_qkv"][i] for i in range(3)], [qkv[i] for i in range(3)])
        attn, actx = self.attn.forward(qkv[0], qkv[1], qkv[2])
        S.update(a_qkv=a_qkv, qkv=qkv, attn=attn, actx=actx)

    # ------------------------------------------------------------------ backward pieces
    @_nvtx
    def _up_bwd(self, names, dgrad_probs, wgrad_pairs, da_P, zP, s, dss_name):
        """Backward of one chunk boundary: dgrad of the up-projection(s) into da_P, then the rank-r
        all-reduce of da_P started asynchronously (NCCL's stream) while the independent weight
        gradient GEMM runs, then sigma-bwd (+ norm-bwd prologue) in place once the sum landed.
        zP is the stored z (= all-reduce buffer of the forward): [T, k*r] grouped, [k, T, r] not."""
        if self.peer is not None:
            return self._up_bwd_peer(names, dgrad_probs, wgrad_pairs, zP, s, dss_name)
        if (self.grouping or len(dgrad_probs) == 1) and not self.comm.live:
            self._dgrad_wgrad(dgrad_probs, wgrad_pairs)  # no-op collective below: one launch when it fits
            wgrad_pairs = None
        elif self.grouping or len(dgrad_probs) == 1:
            self._gemm(*dgrad_probs)
        else:
            for p in dgrad_probs:
                self._gemm(p)
        k = len(names)
        if self.grouping or k == 1:
            handles = [self.comm.all_reduce_start(da_P, names[0] if k == 1 else self._gid(names))]
        else:
            handles = [self.comm.all_reduce_start(da_P[i], nm) for i, nm in enumerate(names)]
        if wgrad_pairs is not None:
            self._wgrad(wgrad_pairs)
        for h in handles:
            self.comm.wait(h)
        return self._sigma_bwd(names, da_P, zP, s, dss_name)

    def _up_bwd_peer(self, names, dgrad_probs, wgrad_pairs, z_own, s_own, dss_name):
        """dgrad into the symmetric dA -> "ready" -> weight-gradient GEMM (independent, covers the
        peers' arrival) -> ONE kernel: pull-reduce the owned rows of every rank's dA, sigma-bwd +
        normalisation-bwd on them, push dP (and dss) into every rank -> "done"."""
        T, r, k = self.T, self.r, len(names)
        key = "_".join(names)
        pc = self.peer
        if pc.scatter:  # dgrad + reduce-scatter in one kernel, into the owners' RdA buffers
            self._gemm_scatter(*[dataclasses.replace(q, c=None) for q in dgrad_probs], owner_buf=f"RdA_{key}",
                               col0=[i * r for i in range(len(dgrad_probs))])
        else:
            self._gemm(*dgrad_probs)
        pc.signal(peer.READY)
        self._wgrad(wgrad_pairs)
        pc.wait(peer.READY)
        dP = self.buf(f"dP_{key}", (T, k * r))
        dss = self.buf(dss_name, (T,), F32) if s_own is not None else None
        if pc.scatter:
            peer.boundary_bwd_local(pc, f"RdA_{key}", T, k * r, r, self.var, self.d, z_own, s_own, f"dP_{key}",
                                    dss_name if s_own is not None else None)
        else:
            peer.boundary_bwd(pc, f"dA_{key}", T, k * r, r, self.var, self.d, z_own, s_own, f"dP_{key}",
                              dss_name if s_own is not None else None)
        pc.exchange(peer.DONE)
        self.stats.kernel_launches += 5
        self.comm.trace.emit("all-reduce", names[0] if k == 1 else self._gid(names), "block", T * k * r,
                             self.comm.pass_tag)
        return dP, dss

    def _sigma_bwd(self, names, da_P, zP, s, dss_name):
        k, r, T = len(names), self.r, self.T
        out = None
        if self.lax and self.has_h_prev:
            # dL/dh_prev = dL/da (the merge is an add): keep the reduced da, write dP beside it
            out = self.buf(f"dPlax_{'_'.join(names)}", tuple(da_P.shape))
            views = self._da_views(names, da_P)
            if self.dh_prev is None:
                self.dh_prev = {}
            self.dh_prev.update(zip(names, views))
        if self.lax and self.dh_cur_in is not None:
            # h_cur = z also feeds the next layer's merge: dz = da + dL/dh_cur
            key = f"dzlax_{'_'.join(names)}"
            if self.grouping or k == 1:
                dz = self._lax_add(self._da_views(names, da_P), [self.dh_cur_in[n] for n in names], key, names)
            else:
                dz = self.buf(key, (k, T, r))
                for i, n in enumerate(names):
                    K.add(da_P[i], self.dh_cur_in[n], dz[i])
                    self.stats.kernel_launches += 1
            da_P = dz
        if out is None:
            out = da_P  # in place
        if self.grouping or k == 1:
            dss = self.buf(dss_name, (T,), F32) if s is not None else None
            K.fixup_sigma_bwd(zP, da_P, out, r=r, nproj=k, variant=self.var, s=s, d=self.d, dss=dss)
            self.stats.kernel_launches += 1
            return out, dss
        # ungrouped: the norm statistic gradient sums over the projections
        parts = self.buf(f"{dss_name}_parts", (k, 1, T), F32) if s is not None else None
        for i in range(k):
            K.fixup_sigma_bwd(zP[i], da_P[i], out[i], r=r, nproj=1, variant=self.var, s=s, d=self.d,
                              dss=None if parts is None else parts[i, 0])
            self.stats.kernel_launches += 1
        if s is None:
            return out, None
        dss = self.buf(dss_name, (T,), F32)
        K.reduce_rows(parts, dss.view(1, T))
        self.stats.kernel_launches += 1
        return out, dss

    def _da_buffer(self, names):
        T, r, k = self.T, self.r, len(names)
        if self.grouping or k == 1:
            return self.buf(f"dA_{'_'.join(names)}", (T, k * r))
        return self.buf(f"dA3_{'_'.join(names)}", (k, T, r))

    def _da_views(self, names, da):
        r = self.r
        if self.grouping or len(names) == 1:
            return [da[:, i * r:(i + 1) * r] for i in range(len(names))]
        return [da[i] for i in range(len(names))]

    @_nvtx
    def _down_bwd(self, names, dP, W, x_res, gamma, dres, dx_out, dss, grad_key, gamma_key):
        """dh = dP @ W (dgrad) ; dW = (dP^T x) * gamma (wgrad) ; dx = dres + dh*gamma + 2 x dss."""
        T, dl, r, k = self.T, self.dl, self.r, len(names)
        dh = self.buf("dh", (T, dl))
        if self.grouping or k == 1:
            self._dgrad_wgrad([K.Gemm(dP, W, dh, b_mn=True)], [(dP, x_res, self.grad[grad_key])], col_scale=gamma)
        else:
            # dh = sum_i dP_i @ W_i, accumulated through the residual epilogue (one launch each,
            # like the reference's per-projection GEMMs)
            for i in range(k):
                self._gemm(K.Gemm(dP[i], W[i * r:(i + 1) * r], dh, b_mn=True, resid=dh if i else None))
            g = self.grad[grad_key]
            self._wgrad([(dP[i], x_res, g[i * r:(i + 1) * r]) for i in range(k)], col_scale=gamma)
        gparts = self.buf("gparts", (4 * self.sms, dl), F32)
        nb = K.rmsnorm_bwd(dh, x_res, gamma, dss, dx_out, gparts, dres=dres)
        K.reduce_rows(gparts[:nb].view(nb, 1, dl), self.grad[gamma_key].view(1, dl))
        self.stats.kernel_launches += 2

    # ------------------------------------------------------------------ backward
    def backward(self, dy: torch.Tensor) -> torch.Tensor:
        """dy: upstream gradient of this rank's y shard [T, d/tp] bf16. Returns dx shard and fills
        self.grad (fp32) for every local weight."""
        S, W, T, dl, fl, r = self.saved, self.W, self.T, self.dl, self.flp, self.r
        if not S:
            raise RuntimeError("backward called before forward")
        if self.ckpt:
            self._recompute_mlp_inputs()
        self.comm.pass_tag = "backward"
        self.dh_prev = None
        G = self.grad
        # ---------------- mlp down chunk: y = x_mid + a_d @ Wu_d^T
        names = ("down",)
        da = self._da_buffer(names)
        dP, _ = self._up_bwd(names, [K.Gemm(dy, W["u_d"], da, b_mn=True)],    # da_d = dy @ Wu_d
                             [(dy, S["a_d"][0], G["u_d"])],                     # dWu_d = dy^T a_d
                             da, S["P_d"], None, "dss_d")
        gu = S["gu"]
        dgu = self.buf("dgu", (2, T, fl))
        if self.fuse_swiglu_bwd:
            # dact = dz_d @ Wd_d never leaves the GEMM: its epilogue emits dg and du directly
            self._gemm(K.Gemm(dP, W["d_d"], dgu[0], b_mn=True, swiglu_bwd=(gu[0], gu[1], dgu[1])))
        else:
            dact = self.buf("dact", (T, fl))
            self._dgrad_wgrad([K.Gemm(dP, W["d_d"], dact, b_mn=True)],         # dact = dz_d @ Wd_d
                              [(dP, S["act"], G["d_d"])])                       # dWd_d = dz_d^T act
            K.swiglu_bwd(gu[0], gu[1], dact, dgu[0], dgu[1])
            self.stats.kernel_launches += 1
        if self.fuse_swiglu_bwd:
            self._wgrad([(dP, S["act"], G["d_d"])])
        # ---------------- gate|up chunk
        names = ("gate", "up")
        da = self._da_buffer(names)
        dav = self._da_views(names, da)
        dP, dss2 = self._up_bwd(names, [K.Gemm(dgu[i], W["u_gu"][i], dav[i], b_mn=True) for i in range(2)],
                                [(dgu[i], S["a_gu"][i], G["u_gu"][i]) for i in range(2)],
                                da, S["P_gu"], S["s2"], "dss2")
        dx_mid = self.buf("dx_mid", (T, dl))
        self._down_bwd(names, dP, W["d_gu"], S["x_mid"], self.gamma2, dy, dx_mid, dss2, "d_gu", "gamma2")
        # ---------------- attention o chunk: x_mid = x + a_o @ Wu_o^T
        if self.ckpt:
            self._recompute_attn_inputs()
            self.comm.pass_tag = "backward"
        names = ("o",)
        da = self._da_buffer(names)
        dP, _ = self._up_bwd(names, [K.Gemm(dx_mid, W["u_o"], da, b_mn=True)], [(dx_mid, S["a_o"][0], G["u_o"])],
                             da, S["P_o"], None, "dss_o")
        dattn = self.buf("dattn", (T, dl))
        self._dgrad_wgrad([K.Gemm(dP, W["d_o"], dattn, b_mn=True)], [(dP, S["attn"], G["d_o"])])
        dq, dk, dv = self.attn.backward(dattn, S["actx"])
        # ---------------- q|k|v chunk
        names = ("q", "k", "v")
        da = self._da_buffer(names)
        dav = self._da_views(names, da)
        dqkv = (dq, dk, dv)
        dP, dss1 = self._up_bwd(names, [K.Gemm(dqkv[i], W["u_qkv"][i], dav[i], b_mn=True) for i in range(3)],
                                [(dqkv[i], S["a_qkv"][i], G["u_qkv"][i]) for i in range(3)],
                                da, S["P_qkv"], S["s1"], "dss1")
        dx = self.buf("dx", (T, dl))
        self._down_bwd(names, dP, W["d_qkv"], S["x"], self.gamma1, dx_mid, dx, dss1, "d_qkv", "gamma1")
        self._join_side()
        return dx
