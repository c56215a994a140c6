"""Public entry points, drop-in for the reference's `execute_forward` (simulator.py:268-316)
plus the training step the reference does not have.

Process model: one process per GPU. At tp == 1 no process group is needed. At tp > 1 the
caller runs one process per TP rank with torch.distributed initialised (NCCL on the box); each
rank calls the same function with the same logical inputs, exactly like the reference's SPMD
ranks, and gets back the same gathered logical output.

Input/output convention matches the reference: x is a host `Tensor` [b, s, d] (float64 values),
y is returned as a host float64 `Tensor` [b, s, d]. Arithmetic runs in bf16/fp32 on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .comm import TPComm
from .executor import BTPBlockExecutor
from .interop import as_block, as_h_prev, as_plan, element_bytes_of, values_of
from .model import EPS_DEFAULT, DecoderBlockWeights, Variant
from .plan import PlanError, ShardPlan, Strategy, plan
from .tensor import Tensor
from .trace import Trace

BF16 = torch.bfloat16


@dataclass
class SimResult:
    """Same fields as the reference's SimResult (simulator.py:189-195). `workspaces` holds only
    THIS rank's dict (index rank) — other ranks live in other processes — and is filled only
    when capture_workspaces=True."""

    y: Tensor
    h_cur: dict | None
    trace: Trace
    workspaces: list
    plan: ShardPlan


@dataclass
class StepResult:
    y: Tensor
    loss: float
    dx: np.ndarray            # this rank's [T, d/tp] input-gradient shard (float64 host copy)
    grads: dict               # this rank's weight grads keyed like the reference block
    trace: Trace
    plan: ShardPlan
    executor: object
    h_cur: dict | None = None     # lax: {projection: Tensor [b, s, r]} (the bundle for the next layer)
    dh_prev: dict | None = None   # lax with an h_prev: {projection: dL/dh_prev [b, s, r]} (float64 host)


def _normalise(pl, block):
    """Our plan / block for ours or the reference's own objects (interop.py). block=None: the
    caller supplies its own executor (ModelTrainer)."""
    return as_plan(pl), None if block is None else as_block(block)


def _check_inputs(pl: ShardPlan, block: DecoderBlockWeights, x) -> np.ndarray:
    if block.variant is not pl.variant:
        raise PlanError(f"plan variant {pl.variant.value} != block variant {block.variant.value}")
    xv = values_of(x)
    if xv.ndim != 3 or xv.shape[2] != pl.cfg.d:
        raise PlanError(f"x must be [b, s, d={pl.cfg.d}], got {tuple(xv.shape)}")
    if (xv.shape[0], xv.shape[1]) != (pl.shape.b, pl.shape.s):
        raise PlanError(f"x batch/seq {tuple(xv.shape[:2])} disagrees with plan shape")
    return xv


def make_executor(pl: ShardPlan, block: DecoderBlockWeights, *, eps: float = EPS_DEFAULT, trace: Trace | None = None,
                  device=None, attn_backend: str = "auto", precision: str = "bf16", comm: TPComm | None = None,
                  boundary: str = "nccl", peer_provider: str = "symmetric_memory", boundary_dtype: str = "bf16"):
    """Build this rank's executor for the plan's strategy (comm: default = the process group).

    boundary_dtype="fp32" (BTP, NCCL boundaries): the forward rank-r all-reduces carry an fp32
    partial (one bf16 rounding of the cross-rank sum instead of one per ring hop; 2x the bytes).

    boundary="peer" (BTP, tp > 1): the chunk boundaries run as fused reduce-scatter -> fix-up/sigma
    -> all-gather kernels over NVLink peer memory (torch symmetric-memory heap, csrc/peer.cu)
    instead of NCCL all-reduces + a fix-up launch. boundary="nvls": the same kernels' NVLink-SHARP
    form — the switch reduces the partials (multimem.ld_reduce) and replicates the results
    (multimem.st) through the heap's multicast mapping. peer_provider: how the ranks' heaps are
    mapped — "symmetric_memory" (torch), or "cuda_ipc" (cudaIpc handles over the process group)."""
    if boundary not in ("nccl", "peer", "nvls"):
        raise ValueError(f"boundary must be 'nccl', 'peer' or 'nvls', got {boundary!r}")
    if boundary_dtype not in ("bf16", "fp32"):
        raise ValueError(f"boundary_dtype must be 'bf16' or 'fp32', got {boundary_dtype!r}")
    pl, block = _normalise(pl, block)
    if comm is None:
        comm = TPComm.from_env(pl.shape.tp, trace=trace if trace is not None else Trace())
        if boundary in ("peer", "nvls") and pl.strategy is Strategy.BOTTLENECK:
            from .peer import PeerComm

            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            comm = TPComm(comm.tp, comm.rank, comm.group, comm.trace,
                          peer=PeerComm(comm.tp, comm.rank, dev, provider=peer_provider,
                                        nvls=boundary == "nvls"))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if pl.strategy is Strategy.BOTTLENECK:
        ex = BTPBlockExecutor(pl, block, comm, dev, eps, attn_backend, precision)
        ex.boundary_dtype = boundary_dtype
        return ex
    from .baselines import FullRankExecutor, VanillaExecutor

    cls = VanillaExecutor if pl.strategy is Strategy.VANILLA else FullRankExecutor
    return cls(pl, block, comm, dev, eps, attn_backend, precision)


def shard_input(ex, xv: np.ndarray) -> torch.Tensor:
    """This rank's slice of the logical input as a device bf16 [T, width] tensor."""
    T = xv.shape[0] * xv.shape[1]
    x2 = xv.reshape(T, -1)
    if getattr(ex, "residual_sharded", True):
        lo = ex.rank * ex.dl
        x2 = x2[:, lo:lo + ex.dl]
    return torch.from_numpy(np.ascontiguousarray(x2)).to(ex.dev, ex.act)


def _gather_y(ex, y_sh: torch.Tensor, model_tail: bool) -> torch.Tensor:
    if not getattr(ex, "residual_sharded", True):
        return y_sh
    if model_tail:
        return ex.comm.all_gather_cols(y_sh, "final-gather", tag="boundary")
    if not ex.comm.live:
        return y_sh if ex.tp == 1 else y_sh.repeat(1, ex.tp)
    # host-side result assembly (the reference concatenates without a record, simulator.py:713)
    parts = [torch.empty_like(y_sh) for _ in range(ex.tp)]
    dist.all_gather(parts, y_sh.contiguous(), group=ex.comm.group)
    return torch.cat(parts, dim=1)


def execute_forward(pl: ShardPlan, block: DecoderBlockWeights, x, h_prev=None, *, eps: float = EPS_DEFAULT,
                    model_tail: bool = False, trace: Trace | None = None, capture_workspaces: bool = False,
                    attn_backend: str = "auto", precision: str = "bf16") -> SimResult:
    """Run one block forward under the plan on the GPU; returns the gathered logical y (and, for
    lax, the h_cur bundle; h_prev is given logically, {projection: Tensor [b, s, r]}, as in the
    reference simulator.py:268-316). pl / block / x / h_prev may be the reference's own objects."""
    pl, block = _normalise(pl, block)
    xv = _check_inputs(pl, block, x)
    ex = make_executor(pl, block, eps=eps, trace=trace, attn_backend=attn_backend, precision=precision)
    _stage_h_prev(ex, block, h_prev)
    x_sh = shard_input(ex, xv)
    y_sh = ex.forward(x_sh)
    y = _gather_y(ex, y_sh, model_tail)
    ws = [dict() for _ in range(pl.shape.tp)]
    if capture_workspaces:
        ws[ex.rank] = ex.capture_workspaces()
    b, s, d = xv.shape
    y_host = y.double().cpu().numpy().reshape(b, s, d)
    eb = element_bytes_of(x)
    return SimResult(Tensor(y_host, eb), _h_cur(ex, b, s, eb), ex.comm.trace, ws, pl)


def reference_forward(block: DecoderBlockWeights, x, h_prev=None, eps: float = EPS_DEFAULT, *,
                      precision: str = "fp32"):
    """Single-device forward of one block (reference model.py:256-305) on the GPU: a TP = 1 plan of
    the block's own variant (BTP for low-rank blocks, Megatron for full-rank; at one rank both
    are the plain block). Returns (y Tensor [b, s, d], h_cur bundle for lax else None).
    precision="fp32" (default) keeps it within the north_star 1e-4 of the float64 reference."""
    from .model import RunShape

    block = as_block(block)
    xv = values_of(x)
    if xv.ndim != 3 or xv.shape[2] != block.cfg.d:
        from .tensor import DimensionError

        raise DimensionError(f"x must be [b, s, d={block.cfg.d}], got {tuple(xv.shape)}")
    b, s, _ = xv.shape
    if block.variant is Variant.FULL_RANK:
        pl = plan(Strategy.FULL_RANK, block.cfg, RunShape(b, s, 1))
    else:
        pl = plan(Strategy.BOTTLENECK, block.cfg, RunShape(b, s, 1), block.variant, online_norm=True, grouping=True)
    res = execute_forward(pl, block, x, h_prev, eps=eps, precision=precision)
    return res.y, res.h_cur


def _stage_h_prev(ex, block: DecoderBlockWeights, h_prev) -> None:
    if block.variant is not Variant.LAX:
        return  # the reference ignores a bundle handed to a non-lax block (simulator.py:297)
    if h_prev is not None:
        h_prev = {k: values_of(v) for k, v in h_prev.items()}
    ex.set_h_prev(h_prev)


def _bundle_host(ex, views: dict, b, s) -> dict:
    """{projection: float64 [b, s, r]} from device views: replicated under BTP (read this rank's),
    r-sliced per rank under naive TP (gathered; lax slices are contiguous, simulator.py:440-447)."""
    out = {}
    for n, h in views.items():
        if not getattr(ex, "residual_sharded", True) and ex.tp > 1:
            if ex.comm.live:
                parts = [torch.empty_like(h.contiguous()) for _ in range(ex.tp)]
                dist.all_gather(parts, h.contiguous(), group=ex.comm.group)
                h = torch.cat(parts, dim=1)
            else:
                h = h.repeat(1, ex.tp)
        out[n] = h.double().cpu().numpy().reshape(b, s, -1)
    return out


def _h_cur(ex, b, s, eb=2):
    """The lax bundle {projection: Tensor [b, s, r]} for the next layer, else None."""
    if not getattr(ex, "lax", False):
        return None
    torch.cuda.synchronize(ex.dev)
    return {n: Tensor(v, eb) for n, v in _bundle_host(ex, ex.h_cur, b, s).items()}


def train_step(pl: ShardPlan, block: DecoderBlockWeights, x, G=None, *, eps: float = EPS_DEFAULT,
               attn_backend: str = "auto", executor=None, precision: str = "bf16", h_prev=None) -> StepResult:
    """Forward + backward of the block for the builder-defined loss L = sum(y * G) (dL/dy = G).
    lax: h_prev ({projection: [b, s, r]}) is merged after each reduction; the result carries the
    h_cur bundle and dL/dh_prev.

    G defaults to the loss projection seeded_fill((b, s, d), 30000)."""
    from .tensor import seeded_fill

    pl, block = _normalise(pl, block)
    xv = _check_inputs(pl, block, x)
    b, s, d = xv.shape
    if G is None:
        G = seeded_fill((b, s, d), 30000).values
    Gv = values_of(G)
    ex = executor if executor is not None else make_executor(pl, block, eps=eps, attn_backend=attn_backend,
                                                             precision=precision)
    _stage_h_prev(ex, block, h_prev)
    x_sh = shard_input(ex, xv)
    g_sh = shard_input(ex, Gv)
    y_sh = ex.forward(x_sh)
    h_cur = _h_cur(ex, b, s)
    loss = ex.loss(y_sh, g_sh)
    dx = ex.backward(g_sh)
    y = _gather_y(ex, y_sh, False)
    dh = getattr(ex, "dh_prev", None)
    dh_host = None if dh is None else _bundle_host(ex, dh, b, s)
    return StepResult(
        y=Tensor(y.double().cpu().numpy().reshape(b, s, d)),
        loss=loss,
        dx=dx.double().cpu().numpy(),
        grads=ex.weight_grads_by_name(),
        trace=ex.comm.trace,
        plan=pl,
        executor=ex,
        h_cur=h_cur,
        dh_prev=dh_host,
    )


class BlockTrainer:
    """Persistent block training step on this rank: weights, activations and workspaces stay
    resident in HBM; one step = forward + loss + backward + fused AdamW update of this rank's
    parameter shard (fp32 master weights and moments; `optimizer=False` drops the update). At tp == 1 the whole step is captured
    once into a CUDA graph and replayed (the step is ~60 kernel launches).

    step_device(x, G): device-resident inputs, no host sync (the bench's `value`).
    step(x_host, G_host): the user-facing call — H2D copy of this step's pinned-host inputs,
    the step, and a D2H read of the loss.
    fit(x_hosts, G_host): the training loop — the loss projection G is copied once, each batch's
    pinned-host x is copied on a side stream while the previous step computes (two input slots,
    one CUDA graph each), and every step's loss is read back (the bench's `e2e`)."""

    def __init__(self, pl: ShardPlan, block: DecoderBlockWeights, *, eps: float = EPS_DEFAULT,
                 attn_backend: str = "auto", use_graph: bool = True, adamw: dict | None = None,
                 optimizer: bool = True, comm: TPComm | None = None, executor=None, boundary: str = "nccl",
                 graph_collectives: bool = True, peer_provider: str = "symmetric_memory",
                 boundary_dtype: str = "bf16"):
        pl, block = _normalise(pl, block)
        self.pl = pl
        self.ex = executor if executor is not None else make_executor(pl, block, eps=eps, attn_backend=attn_backend,
                                                                      comm=comm, boundary=boundary,
                                                                      peer_provider=peer_provider,
                                                                      boundary_dtype=boundary_dtype)
        # AdamW hyper-parameters (lr, b1, b2, eps, wd); the update is part of every step unless disabled
        self.adamw = dict(adamw or {}) if optimizer else None
        # A step without live collectives is always graphed. With live NCCL collectives the whole
        # step (NCCL kernels included) is captured too when graph_collectives — the TP > 1 step is
        # ~100 launches per rank — and falls back to eager launches if the capture is refused.
        live = self.ex.comm.live
        nccl = live and dist.get_backend(self.ex.comm.group) == "nccl"
        self.use_graph = use_graph and (not live or (nccl and graph_collectives))
        self.graphs: dict = {}
        self.graphed = False
        self._per_step_launches = 0
        self._replays = 0
        self._x = self._g = None
        self.loss_buf = None
        self._slots = None
        self._copy_stream = None

    @property
    def kernel_launches(self) -> int:
        return self.ex.stats.kernel_launches + self._replays * self._per_step_launches

    def device_inputs(self, x: np.ndarray, G: np.ndarray):
        self._x, self._g = shard_input(self.ex, np.asarray(x)), shard_input(self.ex, np.asarray(G))
        return self._x, self._g

    def pinned_host_inputs(self, x: np.ndarray, G: np.ndarray):
        xs, gs = shard_input(self.ex, np.asarray(x)).cpu(), shard_input(self.ex, np.asarray(G)).cpu()
        return xs.pin_memory(), gs.pin_memory()

    def _fwd(self, x):
        self._y = self.ex.forward(x)

    def _tail(self, g):
        self.loss_buf = self.ex.loss_device(self._y, g)
        self._dx = self.ex.backward(g)
        if self.adamw is not None:
            self.ex.optimizer_step(**self.adamw)

    def _eager(self, x, g, g_ready=None):
        self._fwd(x)
        if g_ready is not None:
            torch.cuda.current_stream().wait_event(g_ready)
        self._tail(g)

    def step_device(self, x: torch.Tensor, g: torch.Tensor, g_ready=None) -> None:
        """One step on device-resident inputs. g_ready (optional CUDA event): the forward only
        needs x, so the loss-side input g may still be in flight — the stream waits for it between
        the forward and the loss (fit() uses this to hide its one-time G copy behind step 0)."""
        if not self.use_graph:
            self._eager(x, g, g_ready)
            return
        key = (x.data_ptr(), g.data_ptr())
        graphs = self.graphs.get(key)
        if graphs is None:
            # the first step runs eagerly (allocating every buffer); the step is then captured as
            # two graphs — forward, and loss + backward + update (sharing one memory pool) — that
            # later calls replay back to back
            before = self.ex.stats.kernel_launches
            self._eager(x, g, g_ready)
            self._per_step_launches = self.ex.stats.kernel_launches - before
            torch.cuda.synchronize()
            g_fwd, g_tail = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            saved = self.ex.stats.kernel_launches
            n_rec = len(self.ex.comm.trace.records)
            try:
                with torch.cuda.stream(side):
                    with torch.cuda.graph(g_fwd, stream=side):
                        self._fwd(x)
                    with torch.cuda.graph(g_tail, stream=side, pool=g_fwd.pool()):
                        self._tail(g)
            except Exception as exc:  # capture refused (e.g. a backend without graph support): stay eager
                import warnings

                warnings.warn(f"CUDA-graph capture of the training step failed ({exc}); running eagerly")
                torch.cuda.synchronize()
                self.use_graph = False
                return
            finally:
                self.ex.stats.kernel_launches = saved
                del self.ex.comm.trace.records[n_rec:]  # a capture issues no collectives
            torch.cuda.current_stream().wait_stream(side)
            self.graphs[key], self.graphed = (g_fwd, g_tail), True
            return
        g_fwd, g_tail = graphs
        g_fwd.replay()
        if g_ready is not None:
            torch.cuda.current_stream().wait_event(g_ready)
        g_tail.replay()
        self._replays += 1

    FIRST_COPY_STREAMS = 4  # copy streams for the first batch's (exposed) H2D in fit()

    def fit(self, x_hosts, G_host: torch.Tensor) -> list[float]:
        """Pipelined steps over pinned-host input shards; returns every step's loss.

        Every step's loss is copied device->host (4 bytes into a pinned ring) right behind the
        step on the compute stream, and the host reads it one step later, after it has already
        queued the next step, so the GPU never idles on the host's read-back round trip."""
        dev = self.ex.dev
        if self._slots is None:
            shape, dt = x_hosts[0].shape, x_hosts[0].dtype
            self._slots = [torch.empty(shape, dtype=dt, device=dev) for _ in range(2)]
            self._target = torch.empty(G_host.shape, dtype=G_host.dtype, device=dev)
            self._copy_stream = torch.cuda.Stream(device=dev)
            self._first_streams = [torch.cuda.Stream(device=dev) for _ in range(self.FIRST_COPY_STREAMS - 1)]
        main, copy = torch.cuda.current_stream(), self._copy_stream
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
        g_copied = torch.cuda.Event()
        copy.wait_stream(main)
        # the first batch's H2D is the one copy no step hides: it goes out in row slices on several
        # copy streams at once (one 64 MiB pinned copy: 36 GB/s on one stream, 48 GB/s on four,
        # scripts/probe_h2d.py); later batches copy on one stream under the previous step
        n_sl = len(self._first_streams) + 1
        rows = x_hosts[0].shape[0]
        if n_sl > 1 and rows % n_sl == 0:
            step = rows // n_sl
            joins = []
            for j, st in enumerate([copy] + self._first_streams):
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    self._slots[0][j * step:(j + 1) * step].copy_(x_hosts[0][j * step:(j + 1) * step], non_blocking=True)
                    if j:
                        ev = torch.cuda.Event()
                        ev.record(st)
                        joins.append(ev)
            for ev in joins:
                copy.wait_event(ev)
        else:
            with torch.cuda.stream(copy):
                self._slots[0].copy_(x_hosts[0], non_blocking=True)
        with torch.cuda.stream(copy):
            copied[0].record(copy)
            # G (the loss projection) is needed only after step 0's forward: its copy runs under it
            self._target.copy_(G_host, non_blocking=True)
            g_copied.record(copy)
        if getattr(self, "_loss_host", None) is None:
            self._loss_host = torch.zeros(2, dtype=torch.float32).pin_memory()
        read = [torch.cuda.Event(), torch.cuda.Event()]
        losses = []
        for i in range(len(x_hosts)):
            s = i & 1
            main.wait_event(copied[s])
            if i + 1 < len(x_hosts):
                ns = s ^ 1
                if i >= 1:
                    copy.wait_event(consumed[ns])  # slot ns was read by step i-1
                with torch.cuda.stream(copy):
                    self._slots[ns].copy_(x_hosts[i + 1], non_blocking=True)
                    copied[ns].record(copy)
            self.step_device(self._slots[s], self._target, g_ready=g_copied if i == 0 else None)
            consumed[s].record(main)
            self._loss_host[s:s + 1].copy_(self.loss_buf.view(1), non_blocking=True)  # D2H, this step
            read[s].record(main)
            if i >= 1:  # the previous step's loss, read while this step runs
                read[s ^ 1].synchronize()
                losses.append(float(self._loss_host[s ^ 1]))
        if x_hosts:
            last = (len(x_hosts) - 1) & 1
            read[last].synchronize()
            losses.append(float(self._loss_host[last]))
        return losses

    def step(self, x_host: torch.Tensor, g_host: torch.Tensor) -> float:
        if self._x is None:
            self._x = torch.empty(x_host.shape, dtype=x_host.dtype, device=self.ex.dev)
            self._g = torch.empty(g_host.shape, dtype=g_host.dtype, device=self.ex.dev)
        self._x.copy_(x_host, non_blocking=True)
        self._g.copy_(g_host, non_blocking=True)
        self.step_device(self._x, self._g)
        return float(self.loss_buf.item())

    def time_gemms(self, x: torch.Tensor, g: torch.Tensor) -> dict:
        """One step with every GEMM launch bracketed by CUDA events on its stream. The step is
        captured into a CUDA graph (events as record nodes) and replayed, so each interval is
        device time only — no host enqueue gaps. The weight-gradient GEMMs run serialised here
        (not on their side stream), so each interval is one kernel's own duration."""
        execs = [self.ex] + list(getattr(self.ex, "blocks", []))
        saved_cc = [e.concurrent_wgrad for e in execs]
        for e in execs:
            e.concurrent_wgrad = False
        try:
            return self._time_gemms(x, g)
        finally:
            for e, c in zip(execs, saved_cc):
                e.concurrent_wgrad = c

    def _attns(self):
        return [e.attn for e in [self.ex] + list(getattr(self.ex, "blocks", [])) if getattr(e, "attn", None) is not None]

    def _time_gemms(self, x: torch.Tensor, g: torch.Tensor) -> dict:
        self.ex.gemm_timer = []
        for a in self._attns():
            a.timer = None
        self._eager(x, g)  # allocate every buffer outside the capture
        torch.cuda.synchronize()
        if self.ex.comm.live and not self.use_graph:  # collectives eager; timings then include host gaps
            rec, self.ex.gemm_timer = self.ex.gemm_timer, None
            return self._gemm_summary(rec)
        # live NCCL collectives are captured with the step (as in step_device), so every
        # interval is device time only at TP > 1 too
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        saved = self.ex.stats.kernel_launches
        n_rec = len(self.ex.comm.trace.records)
        try:
            with torch.cuda.stream(side):
                self.ex.gemm_timer = []
                attn_rec: list = []
                for a in self._attns():
                    a.timer = attn_rec
                with torch.cuda.graph(graph, stream=side):
                    self._eager(x, g)
        finally:
            self.ex.stats.kernel_launches = saved
            del self.ex.comm.trace.records[n_rec:]
            for a in self._attns():
                a.timer = None
        torch.cuda.current_stream().wait_stream(side)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
        rec, self.ex.gemm_timer = self.ex.gemm_timer, None
        out = self._gemm_summary(rec)
        out["attention_ms"] = {k: sum(a.elapsed_time(b) for a, b, kind in attn_rec if kind == k) for k in ("fwd", "bwd")}
        out["back_to_back"] = self._time_gemm_sequence(x, g)
        return out

    def _time_gemm_sequence(self, x: torch.Tensor, g: torch.Tensor, reps: int = 5) -> dict:
        """The step's GEMM launches alone, in step order on the step's own buffers, captured into
        one graph and replayed back to back between two CUDA events: each launch's device time
        without the per-launch event nodes (which add their own gaps inside a graph). Overwrites
        activations / gradients of the last step — instrumentation only, after the timed region."""
        self.ex.gemm_log = []
        try:
            self._eager(x, g)
        finally:
            log, self.ex.gemm_log = self.ex.gemm_log, None
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                for probs, _ in log:
                    K.gemm(*probs)
        torch.cuda.current_stream().wait_stream(side)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = sum(f for _, f in log)
        return {"ms": ms, "flops": fl, "tflops": fl / (ms / 1e3) / 1e12 if ms else 0.0, "launches": len(log)}

    @staticmethod
    def _gemm_summary(rec) -> dict:
        ms = sum(a.elapsed_time(b) for a, b, _, _ in rec)
        fl = sum(f for _, _, f, _ in rec)
        per = [{"us": a.elapsed_time(b) * 1e3, "tflops": f / (a.elapsed_time(b) / 1e3) / 1e12, "problems": sh}
               for a, b, f, sh in rec]
        return {"ms": ms, "flops": fl, "tflops": fl / (ms / 1e3) / 1e12 if ms else 0.0, "launches": len(rec),
                "per_launch": per}


class ModelTrainer(BlockTrainer):
    """The same persistent, graph-replayed training step for the multi-layer model
    (model_executor.ModelExecutor): inputs are int32 token ids and next-token targets [T]
    (replicated on every TP rank); the loss is the mean cross-entropy of the replicated head."""

    def __init__(self, pl: ShardPlan, mw, *, eps: float = EPS_DEFAULT, attn_backend: str = "auto",
                 use_graph: bool = True, adamw: dict | None = None, optimizer: bool = True,
                 comm: TPComm | None = None, boundary: str = "nccl", peer_provider: str = "symmetric_memory"):
        from .model_executor import ModelExecutor

        if boundary not in ("nccl", "peer", "nvls"):
            raise ValueError(f"boundary must be 'nccl', 'peer' or 'nvls', got {boundary!r}")
        if comm is None:
            comm = TPComm.from_env(pl.shape.tp, trace=Trace())
            if boundary != "nccl" and comm.tp > 1:
                from .peer import PeerComm

                dev = torch.device("cuda", torch.cuda.current_device())
                comm = TPComm(comm.tp, comm.rank, comm.group, comm.trace,
                              peer=PeerComm(comm.tp, comm.rank, dev, provider=peer_provider, nvls=boundary == "nvls"))
        ex = ModelExecutor(pl, mw, comm, torch.device("cuda", torch.cuda.current_device()), eps, attn_backend)
        super().__init__(pl, None, use_graph=use_graph, adamw=adamw, optimizer=optimizer, executor=ex)

    # one step's input is the packed int32 [2, T] (ids, targets): fit() then streams both per batch;
    # the second returned tensor only satisfies the block trainer's (x, G) calling convention
    @staticmethod
    def _pack(ids, targets) -> torch.Tensor:
        return torch.as_tensor(np.stack([np.asarray(ids), np.asarray(targets)]), dtype=torch.int32)

    def device_inputs(self, ids: np.ndarray, targets: np.ndarray):
        self._x = self._pack(ids, targets).to(self.ex.dev)
        self._g = self._x[1]
        return self._x, self._g

    def pinned_host_inputs(self, ids: np.ndarray, targets: np.ndarray):
        packed = self._pack(ids, targets).pin_memory()
        return packed, packed[1]
