#!/usr/bin/env python
"""Benchmark: train tokens/s (fwd+bwd) of one CoLA decoder block under BTP, TP = number of GPUs.

Workload (BASELINE.json configs[1]): CoLA-1B block (d=2048, d_ff=5472, r=512, 32 heads),
b=4, s=4096 (T=16384 tokens per step, counted once per TP group), BTP + online RMSNorm +
grouped GEMMs, cola crossgate, bf16 storage / fp32 accumulation, synthetic seeded inputs and
fan-in-scaled random-init weights. One step = forward + loss + backward (all weight grads).

    python bench.py [--gpus N --steps K --warmup W]           # our arm (TP = N)
    python bench.py --impl reference [...]                     # CPU reference arm (oracle port)
    torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1: one rank per GPU, NCCL

    python bench.py --gpus N ...                               # same: self-launches N ranks via torch.distributed.run

Timing: W warm-up steps, then exactly K steps between barrier + synchronize, CUDA events on the
launching stream, max over ranks. Working set (~1.3 GB of activations) >> L2 (126 MB), so no
L2 flush is needed. Prints ONE JSON line on rank 0 with, beside the contract keys:
  roofline      the tcgen05 GEMM family, per-launch CUDA events inside a replayed graph
  baselines     the same kernels under naive low-rank TP and full-rank Megatron TP (same N, shape,
                step), and BTP's speed-up over each (north_star targets 1.8x / 1.4x at TP=8)
  comm          (N > 1) the plan's boundary all-reduces timed standalone: NCCL bus GB/s vs 900
  cpu_baseline  the oracle port on rank 0's host cores (+ `reference_itself`: btpsim's own
                forward at config C1 when baseline/_ref is installed)
`--dry-run` (CPU, gloo) exercises the launch path and the line's schema without a GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


METRIC = "train tokens/s (fwd+bwd) for CoLA block at TP 1/2/4/8; % of bf16 tensor peak"
UNIT = "tokens/s"
# optimizer update inside every timed step (both arms)
ADAMW = dict(lr=1e-4, b1=0.9, b2=0.95, eps=1e-8, wd=0.1)


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def flops_per_step(cfg, b, s, lowrank=True):
    """Algorithmic FLOPs of one block fwd+bwd: 3*[2T(11dr+3d_ff r) + 4 b s^2 d]."""
    T = b * s
    lin = 2 * T * (11 * cfg.d * cfg.r + 3 * cfg.d_ff * cfg.r) if lowrank else 2 * T * (4 * cfg.d**2 + 3 * cfg.d * cfg.d_ff)
    return 3 * (lin + 4 * b * s * s * cfg.d)


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every 10 ms (a timed
    region of ten ~5 ms steps still gets several samples), else nvidia-smi every 200 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: sw_power_cap 0x4, hw_slowdown 0x8, sw_thermal 0x20, hw_thermal 0x40
    _BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4))

    def __init__(self, index: int = 0):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvidia-smi"
        # NVML is initialised here, before the timed region: nvmlInit can take longer than a whole
        # ten-step region, which then went unsampled
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self._nvml = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), get_reasons)
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self) -> bool:
        pynvml, h, mx, get_reasons = self._nvml
        try:
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = get_reasons(h)
        except Exception:
            return False
        flags = ["Active" if bits & b else "Not Active" for _, b in self._BITS]
        self.rows.append([str(self.index), str(sm), str(mx), "", hex(bits)] + flags)
        return True

    def _run_nvml(self) -> bool:
        if self._nvml is None:
            return False
        while not self._stop.is_set():
            if not self._sample_nvml():
                break
            self._stop.wait(0.01)
        return True

    def _run(self):
        if self._run_nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                return
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


# ------------------------------------------------------------------------------------- CPU arm
def attention_label(attn: str, cfg, args) -> str:
    from paper_2512_12131_b200 import attention as A

    if attn == "auto":
        attn = A.auto_backend(args.s, cfg.d // cfg.heads)
    if attn == "native":
        return "own tcgen05/TMEM flash kernels (btp_attn_fwd / btp_attn_bwd; not a changed subsystem)"
    if attn == "hybrid":
        return "cuDNN SDPA forward + own tcgen05/TMEM backward (btp_attn_bwd; not a changed subsystem)"
    return "cuDNN SDPA via torch (not a changed subsystem)"


def _attention_ab(b, s, h, hd, reps=10):
    """Forward / backward device time of the attention at the step's shape: our kernels
    (btp_attn_fwd / btp_attn_bwd on the [T, h*hd] buffers) vs cuDNN SDPA (the step's default path),
    median of 3 x `reps` back-to-back calls between CUDA events."""
    import math

    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2512_12131_b200 import attention as A
    from paper_2512_12131_b200 import kernels as K

    if not A.native_supported(s, hd):
        return {"skipped": f"native kernels need s % 128 == 0 and hd in (64, 128); s={s}, hd={hd}"}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        out = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) / reps)
        return sorted(out)[1]

    T, W = b * s, h * hd
    gen = torch.Generator(device="cuda").manual_seed(1)
    q, k, v, do = (torch.randn(T, W, device="cuda", generator=gen).bfloat16() for _ in range(4))
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    lse, D = (torch.empty(b, h, s, device="cuda") for _ in range(2))
    acc = torch.empty(T, W, device="cuda")
    nat_f = timed(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
    nat_b = timed(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
    v4 = [t.view(b, s, h, hd).transpose(1, 2).detach().requires_grad_() for t in (q, k, v)]
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        cud_f = timed(lambda: F.scaled_dot_product_attention(*v4, scale=1 / math.sqrt(hd)))
        ref = F.scaled_dot_product_attention(*v4, scale=1 / math.sqrt(hd))
        do4 = do.view(b, s, h, hd).transpose(1, 2)
        cud_b = timed(lambda: torch.autograd.grad(ref, v4, do4, retain_graph=True))
    ref = ref.detach()
    err = float((o.float() - ref.transpose(1, 2).reshape(T, W).float()).norm() / ref.float().norm())
    flops = 4 * b * h * s * s * hd
    return {"shape": {"b": b, "s": s, "heads": h, "head_dim": hd},
            "native": {"fwd_ms": nat_f, "bwd_ms": nat_b, "fwd_tflops": flops / nat_f / 1e9,
                       "bwd_tflops": 2.5 * flops / nat_b / 1e9, "kernels": "btp_attn_fwd / btp_attn_bwd (csrc/attn.cu)"},
            "cudnn": {"fwd_ms": cud_f, "bwd_ms": cud_b, "fwd_tflops": flops / cud_f / 1e9,
                      "bwd_tflops": 2.5 * flops / cud_b / 1e9},
            "native_vs_cudnn_out_rel_err": err,
            "note": "default step (--attn auto at hd 64): cuDNN forward + own backward ('hybrid'); --attn native / "
                    "cudnn run one implementation both ways; profiles/attention/README.md"}


def cpu_oracle_rate(cfg, s, seconds_budget=30.0, max_steps=None, lean=True, optimizer=True):
    """Oracle port (float64 NumPy, BLAS) fwd+bwd+AdamW on a bounded sample: ONE sequence (b=1) of the
    workload's length s. Returns (tokens_per_s, per-step seconds list, threads)."""
    from oracle import btp_oracle as O

    blk = O.build_block(cfg.d, cfg.d_ff, cfg.r, "cola", 0, scale_fan_in=3.0)
    x = O.seeded_fill((s, cfg.d), 10000)
    G = O.loss_projection((s, cfg.d), 30000)
    times, state = [], {}
    with _all_host_threads():
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            y, cache = O.block_forward(blk, x, 1, s, cfg.heads, lean=lean)
            grads = O.block_backward(blk, cache, G, 1, s, cfg.heads)
            if optimizer:
                O.adamw_step(blk, grads, state, **ADAMW)
            times.append(time.perf_counter() - t0)
            if max_steps is not None and len(times) >= max_steps:
                break
            if max_steps is None and time.perf_counter() - t_start > seconds_budget:
                break
        threads = _blas_threads()
    return s / statistics.median(times), times, threads


class _all_host_threads:
    """BLAS on every host thread for the CPU arm, also under torchrun (which exports
    OMP_NUM_THREADS=1 to each rank): the same core count at every N. The CPU arm runs on rank 0
    after the timed GPU work, while the other ranks wait."""

    def __enter__(self):
        self._ctl = None
        try:
            from threadpoolctl import threadpool_limits

            self._ctl = threadpool_limits(limits=os.cpu_count(), user_api="blas")
        except Exception:
            pass
        return self

    def __exit__(self, *exc):
        if self._ctl is not None:
            self._ctl.restore_original_limits()


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # W untimed + K timed steps of the bounded sample (1 sequence of s tokens, fwd+bwd)
    from oracle import btp_oracle as O  # noqa: F401

    # one untimed warm-up sample is enough for the CPU port (BLAS threads spun up, pages touched);
    # each sample is ~10 s of host compute, so W more would only stretch the run
    cpu_oracle_rate(cfg, args.s, max_steps=1)
    rate, times, threads = cpu_oracle_rate(cfg, args.s, max_steps=args.steps)
    ms = statistics.mean(times) * 1e3
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": 1, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"CoLA-{args.config} block fwd+bwd+AdamW, BTP math, b={args.b} s={args.s}",
                   "sample": f"1 sequence x {args.s} tokens per step (b=1 of {args.b})"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"b=1 s={args.s} CoLA-{args.config} block fwd+bwd+AdamW per step, float64 NumPy/BLAS "
                                   "restatement of btpsim (reference itself is forward-only)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.dry_run:
        line["cpu_baseline"]["reference_itself"] = _reference_itself()
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------- GPU arm
def _reduce_max(dist, world, value, dev):
    """Max over ranks of a per-rank scalar (device time: max over ranks)."""
    if world == 1:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class _Timer:
    """CUDA events on the launching (current) stream; perf_counter in --dry-run (no device)."""

    def __init__(self, dry: bool):
        self.dry = dry

    def __enter__(self):
        if self.dry:
            self.t0 = time.perf_counter()
        else:
            import torch

            self.st = torch.cuda.current_stream()
            self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self.e0.record(self.st)
        return self

    def __exit__(self, *exc):
        if self.dry:
            self.ms = (time.perf_counter() - self.t0) * 1e3
        else:
            self.e1.record(self.st)

    def elapsed(self) -> float:
        if self.dry:
            return self.ms
        self.e1.synchronize()
        return self.e0.elapsed_time(self.e1)


class _DryTrainer:
    """--dry-run stand-in for BlockTrainer (CPU, gloo): exercises the launch path, the rendezvous,
    barriers, max-over-ranks timing and the JSON line without a GPU. Never a measurement."""

    def __init__(self, pl):
        import torch

        self.pl, self.graphed, self.kernel_launches = pl, False, 0
        self.w = torch.randn(64, 64)

    def device_inputs(self, x, G):
        import torch

        return torch.as_tensor(x, dtype=torch.float32), torch.as_tensor(G, dtype=torch.float32)

    def pinned_host_inputs(self, x, G):
        return self.device_inputs(x, G)

    def step_device(self, x, g):
        (x.reshape(-1, 64)[:256] @ self.w).sum()

    def fit(self, xs, g):
        for x in xs:
            self.step_device(x, g)
        return [0.0] * len(xs)

    def time_gemms(self, x, g):
        return {"ms": 0.0, "flops": 0.0, "tflops": 0.0, "launches": 0, "per_launch": [],
                "attention_ms": {"fwd": 0.0, "bwd": 0.0}}


def _make_trainer(args, cfg, strategy, shape, comm):
    """The timed object: BlockTrainer (or ModelTrainer with --model) for one TP strategy."""
    from paper_2512_12131_b200.model import Variant, build_block, fan_in_scaled
    from paper_2512_12131_b200.plan import Strategy, plan
    from paper_2512_12131_b200.tensor import seeded_fill

    b, s = shape.b, shape.s
    variant = Variant.FULL_RANK if strategy is Strategy.FULL_RANK else Variant(args.variant)
    pl = plan(strategy, cfg, shape, None if variant is Variant.FULL_RANK else variant,
              online_norm=strategy is Strategy.BOTTLENECK, grouping=not args.no_grouping,
              lowrank_ckpt=args.ckpt and strategy is not Strategy.FULL_RANK)
    if args.dry_run:
        x = seeded_fill((b, s, cfg.d), 10000).values
        return _DryTrainer(pl), pl, variant, x, x
    from paper_2512_12131_b200.api import BlockTrainer

    if args.model:
        # the multi-layer model: embedding shard + L blocks + LM head + cross-entropy
        from paper_2512_12131_b200.api import ModelTrainer
        from paper_2512_12131_b200.model import build_model, token_batch

        if strategy is not Strategy.BOTTLENECK:
            raise SystemExit("--model runs the BTP strategy")
        mw = build_model(cfg, variant, 0, args.vocab, layers=args.layers or cfg.layers)
        x, G = token_batch(b, s, args.vocab)
        trainer = ModelTrainer(pl, mw, use_graph=not args.no_graph, attn_backend=args.attn, adamw=ADAMW,
                               optimizer=not args.no_optimizer, comm=comm, boundary=args.boundary,
                               peer_provider=args.peer_provider)
        return trainer, pl, variant, x, G
    blk = fan_in_scaled(build_block(cfg, variant, 0))
    x = seeded_fill((b, s, cfg.d), 10000).values
    G = seeded_fill((b, s, cfg.d), 30000).values
    boundary = args.boundary if strategy is Strategy.BOTTLENECK else "nccl"
    trainer = BlockTrainer(pl, blk, use_graph=not args.no_graph, attn_backend=args.attn, adamw=ADAMW,
                           optimizer=not args.no_optimizer, comm=comm, boundary=boundary,
                           peer_provider=args.peer_provider,
                           boundary_dtype=args.boundary_dtype if strategy is Strategy.BOTTLENECK else "bf16")
    if variant is Variant.LAX:  # a resident previous-layer bundle, like G (the merge runs every step)
        from paper_2512_12131_b200.model import seeded_h_prev

        trainer.ex.set_h_prev({n: h.values for n, h in seeded_h_prev(cfg, shape, 20000).items()})
    return trainer, pl, variant, x, G


def _time_steps(args, trainer, x_dev, g_dev, barrier, clk=None):
    """W untimed warm-up steps, then exactly K steps between barrier + synchronize; ms per step
    on this rank (the caller takes the max over ranks) and the launches counted in the region."""
    for _ in range(args.warmup):
        trainer.step_device(x_dev, g_dev)
    barrier()
    launches0 = trainer.kernel_launches
    tm = _Timer(args.dry_run)
    if clk is not None:
        clk.__enter__()
    try:
        with tm:
            for _ in range(args.steps):
                trainer.step_device(x_dev, g_dev)
        barrier()
    finally:
        if clk is not None:
            clk.__exit__(None, None, None)
    return tm.elapsed() / args.steps, trainer.kernel_launches - launches0


def _comm_profile(args, pl, comm_tp, world, dist, dev, ms_step):
    """TP > 1: every forward chunk-boundary collective of the plan (`enumerate_collectives`, the
    reference's SimGroup calls simulator.py:123-186) timed standalone through TPComm — the bf16
    [T, k*r] payload and, where the plan has one, its fp32 rider in the same NCCL group — with CUDA
    events, max over ranks. Bus bandwidth = payload bytes * 2(n-1)/n / time (ring all-reduce
    convention, nccl-tests busbw) against NVLink 5's 900 GB/s per direction. The backward mirrors
    each forward boundary (same payload), so per step = 2 x the forward sum; `share_of_step` is
    that un-overlapped sum over the measured step (an upper bound: backward reductions overlap the
    weight-gradient GEMMs)."""
    import torch

    from paper_2512_12131_b200.comm import TPComm
    from paper_2512_12131_b200.plan import enumerate_collectives

    comm = TPComm.from_env()
    dt = torch.float32 if args.dry_run else torch.bfloat16
    rows, reps = [], 20
    for pc in enumerate_collectives(pl):
        if pc.tag != "block" or pc.chunk_id.endswith("-stat"):
            continue
        main = torch.ones(pc.elements, dtype=dt, device=dev)
        rider = torch.ones(dict(pc.extras).get("fused-stat", 0), dtype=torch.float32, device=dev) \
            if pc.extras else None

        def once():
            if rider is not None:
                comm.wait(comm.all_reduce_coalesced_start(main, rider, pc.chunk_id, record=False))
            else:
                comm.wait(comm.all_reduce_start(main, pc.chunk_id, record=False))

        for _ in range(5):
            once()
        if not args.dry_run:
            torch.cuda.synchronize()
        dist.barrier()
        tm = _Timer(args.dry_run)
        with tm:
            for _ in range(reps):
                once()
        ms = _reduce_max(dist, world, tm.elapsed() / reps, dev)
        nbytes = pc.elements * main.element_size() + (0 if rider is None else rider.numel() * 4)
        bus = nbytes * 2 * (world - 1) / world / (ms / 1e3) / 1e9
        rows.append({"chunk": pc.chunk_id, "elements": pc.elements, "rider": 0 if rider is None else rider.numel(),
                     "bytes": nbytes, "us": ms * 1e3, "bus_gbs": bus})
        del main, rider
    fwd_ms = sum(r["us"] for r in rows) / 1e3
    tot_bytes = sum(r["bytes"] for r in rows)
    bus = tot_bytes * 2 * (world - 1) / world / (fwd_ms / 1e3) / 1e9 if fwd_ms else None
    return {"backend": dist.get_backend(), "boundary": args.boundary, "per_boundary_fwd": rows,
            "boundary_ms_per_step": 2 * fwd_ms, "share_of_step": 2 * fwd_ms / ms_step,
            "bus_gbs": bus, "peak_gbs": 900.0, "frac": None if bus is None else bus / 900.0,
            "payload_bytes_per_step": 2 * tot_bytes,
            "note": "standalone NCCL all-reduces of the plan's boundary payloads (bf16 + fp32 rider), "
                    "busbw = bytes*2(n-1)/n/t; share is un-overlapped (upper bound)"}


def _reference_itself():
    """The reference's own forward (btpsim, installed unmodified in baseline/_ref) on config C1:
    execute_forward(plan(BOTTLENECK, CoLA-60M, RunShape(8, 256, 1), COLA, online, grouped),
    build_block(.., 0), x) — SURVEY §8(d). Forward-only: the reference has no backward."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "btpsim").is_dir():
        return {"unavailable": "baseline/_ref (pip --target install of the reference) not present"}
    sys.path.insert(0, str(ref))
    try:
        import btpsim  # noqa: F401
        from btpsim.model import ModelConfig, RunShape, Variant, build_block
        from btpsim.plan import Strategy, plan
        from btpsim.simulator import execute_forward
        from btpsim.tensor import seeded_fill
    finally:
        sys.path.remove(str(ref))
    cfg = ModelConfig(layers=8, heads=8, d=512, d_ff=1376, r=128)
    b, s = 8, 256
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    blk = build_block(cfg, Variant.COLA, 0)
    x = seeded_fill((b, s, cfg.d), 10000)
    t0 = time.perf_counter()
    execute_forward(pl, blk, x)
    sec = time.perf_counter() - t0
    return {"value": b * s / sec, "unit": UNIT, "seconds": sec, "nproc": os.cpu_count(),
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS"), "cores": 1,
            "label": "fwd-only; reference has no backward (btpsim.execute_forward, elementwise NumPy)",
            "config": "C1 CoLA-60M block (d512 d_ff1376 r128 h8) b=8 s=256 TP=1, BTP online grouped"}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        dev = torch.device("cpu")
        if world > 1:
            dist.init_process_group("gloo")
    elif args.share_gpu:
        # debug: every rank on cuda:0, collectives over gloo (the N > 1 code path on a one-GPU box;
        # timings are NOT measurements: the ranks share one GPU and gloo stages through the host)
        local = 0
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        if world > 1:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)

    if not args.dry_run:
        from paper_2512_12131_b200 import executor as _executor

        if args.no_fuse_sigma:
            _executor.FUSE_SIGMA = False
        if args.concurrent_wgrad:
            _executor.ExecutorBase.concurrent_wgrad = True
        if args.no_merge_bwd_gemms:
            _executor.ExecutorBase.merge_bwd_gemms = False
        if args.gemm_pair >= 0:
            from paper_2512_12131_b200 import kernels as _K

            _K.set_pair_mode(args.gemm_pair)
        if args.gemm_st_global >= 0:
            from paper_2512_12131_b200 import kernels as _K

            _K.set_st_global(bool(args.gemm_st_global))
        if args.gemm_res >= 0:
            from paper_2512_12131_b200 import kernels as _K

            _K.set_res4(args.gemm_res)
        if args.attn_bwd_variant >= 0:
            from paper_2512_12131_b200 import _native as _N

            _N.load().btp_attn_tune(3, args.attn_bwd_variant)
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy

    b, s, tp = args.b, args.s, world
    comm = None
    if args.emulate_tp:
        if world != 1:
            raise SystemExit("--emulate-tp runs one rank's share on ONE GPU (no torchrun)")
        from paper_2512_12131_b200.comm import TPComm

        tp = args.emulate_tp
        comm = TPComm.emulated(tp, 0)
    shape = RunShape(b, s, tp)
    strategy = Strategy(args.strategy)

    def barrier():
        if world > 1:
            dist.barrier()
        if not args.dry_run:
            torch.cuda.synchronize()

    trainer, pl, variant, x, G = _make_trainer(args, cfg, strategy, shape, comm)
    x_dev, g_dev = trainer.device_inputs(x, G)
    clk = None if args.dry_run else ClockSampler(local)
    ms, launches = _time_steps(args, trainer, x_dev, g_dev, barrier, clk)
    ms = _reduce_max(dist, world, ms, dev)
    value = b * s / (ms / 1e3)

    # ---- end to end through the public API: pinned host inputs -> H2D -> step -> loss D2H
    # x is the per-step data (two distinct pinned host batches, alternating); G, the fixed loss
    # projection, is copied once per fit() call. Batch i+1's H2D overlaps step i on a side stream.
    xh, gh = trainer.pinned_host_inputs(x, G)
    xh2 = xh.clone().pin_memory() if not args.dry_run else xh.clone()
    trainer.fit([xh, xh2, xh], gh)
    barrier()
    # K steps like the device-timed loop (a longer e2e run measures a hotter GPU: sustained load
    # lowers the SM clock under the power cap; scripts/probe_h2d_interference.py)
    e2e_steps = args.steps
    tm = _Timer(args.dry_run)
    with tm:
        losses = trainer.fit([xh if i % 2 == 0 else xh2 for i in range(e2e_steps)], gh)
    barrier()
    ms_e2e = _reduce_max(dist, world, tm.elapsed() / e2e_steps, dev)
    e2e = {"value": b * s / (ms_e2e / 1e3), "unit": UNIT, "steps": e2e_steps,
           "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
           "d2h_bytes_per_step": 4, "loss": losses[-1], "api": "BlockTrainer.fit (pinned host batches H2D per step on a copy stream; each step's loss copied D2H behind it and read by the host one step later)",
           "h2d_once_per_call_bytes": int(gh.numel() * gh.element_size())}

    # ---- roofline of the dominant kernel (the tcgen05 GEMM family), timed live per launch
    gemm = trainer.time_gemms(x_dev, g_dev)
    if args.dump_gemms and rank == 0:
        Path(args.dump_gemms).write_text(json.dumps(gemm["per_launch"], indent=1))
    peak_burst, peak_sus, hbm, peak_kind = _peaks()
    flops = flops_per_step(cfg, b, s, lowrank=variant is not Variant.FULL_RANK) / tp
    if args.model:  # L blocks (sharded) + the replicated head: 3 * 2 T d V on every rank
        flops = flops * trainer.ex.blocks.__len__() + 3 * 2 * b * s * cfg.d * args.vocab
    traffic, traffic_src = None, None
    b2b = gemm.get("back_to_back") or gemm
    # ncu DRAM bytes of the step's GEMM launches (one capture per launch structure; the newest whose
    # launch count matches this step's, else none)
    for name in ("r02o_gemm_traffic_summary.json", "r02m_gemm_traffic_summary.json", "r02_gemm_traffic_summary.json",
                 "r01_gemm_traffic_summary.json"):
        tfile = ROOT / "profiles" / name
        if not (tfile.exists() and args.config == "1b" and tp == 1 and strategy.value == "btp" and not args.model):
            continue
        t = json.loads(tfile.read_text())
        if t.get("launches") == b2b.get("launches"):
            traffic, traffic_src = t["dram_bytes_per_launch_avg"], t["source"]
            break
    g_ms = b2b["ms"] or float("nan")
    # achieved = the step's GEMM launches replayed back to back (one graph, two CUDA events): each
    # kernel's own device time plus the graph's inter-kernel gap; the per-launch event brackets
    # inside the step graph (event nodes add their own gaps) are reported beside it
    roof = {"bound": "tensor", "kernel": "btp gemm_kernel (all tcgen05 GEMM launches of one step)",
            "achieved": b2b["tflops"], "peak": peak_sus, "unit": "TFLOP/s", "frac": b2b["tflops"] / peak_sus,
            "traffic": traffic, "traffic_unit": "bytes per launch (dram read+write, ncu)", "traffic_source": traffic_src,
            "algorithmic_flops_per_launch": b2b["flops"] / max(b2b["launches"], 1),
            "avg_launch_us": g_ms * 1e3 / max(b2b["launches"], 1),
            "timing": "the step's GEMM launches as one back-to-back graph replay, CUDA events around it",
            "achieved_event_bracketed": gemm["tflops"],
            "peak_kind": f"{peak_kind} sustained bf16 (kernel timed inside a long step)",
            "gemm_share_of_step": g_ms / ms, "gemm_launches_per_step": b2b["launches"],
            "step_frac_of_peak": flops / (ms / 1e3) / 1e12 / peak_sus}
    att = gemm.get("attention_ms", {})
    # where the step goes (device time of one graph-replayed step, kernels serialised): the
    # tcgen05 GEMMs, cuDNN attention (not a changed subsystem), everything else (row kernels, AdamW,
    # collectives, gaps) — a slow run's line says which part moved
    gms = (gemm.get("back_to_back") or gemm)["ms"]
    breakdown = {"gemm_ms": gms, "attention_fwd_ms": att.get("fwd"), "attention_bwd_ms": att.get("bwd"),
                 "other_ms": ms - gms - sum(v for v in att.values() if v)}
    # the attention backward, the step's other large kernel when it is ours (native / hybrid at hd 64):
    # algorithmic FLOPs = its five GEMM-shaped products, 5 x 2 b h s^2 hd, over its in-step time
    roof_att = None
    hd_ = cfg.d // cfg.heads
    from paper_2512_12131_b200.attention import auto_backend

    att_backend = args.attn if args.attn != "auto" else auto_backend(s, hd_)
    if att.get("bwd") and att_backend in ("native", "hybrid"):
        fl_att = 10 * b * (cfg.heads // tp) * s * s * hd_
        ach_att = fl_att / (att["bwd"] * 1e-3) / 1e12
        roof_att = {"bound": "tensor", "kernel": "btp_attn_bwd (D / zero prep + persistent tcgen05 walk + dQ convert)",
                    "achieved": ach_att, "peak": peak_sus, "unit": "TFLOP/s", "frac": ach_att / peak_sus,
                    "algorithmic_flops_per_launch": fl_att, "ms_in_step": att["bwd"],
                    "ceiling": ("hd 64: the N = 64 products (dV, dK, dQ) run at half the M128 tcgen05 rate, so the "
                                "MMA issue floor is ~2160 cycles per (key, query) tile pair, ~0.97 ms at the bench "
                                "shape (~1.4 PF/s, about this measured peak); the exp2 floor (MUFU 16/clk/SM) is "
                                "~0.46 ms (profiles/attention/README.md)")}
    graphed = trainer.graphed
    del trainer, x_dev, g_dev, xh, xh2, gh
    if not args.dry_run:
        torch.cuda.empty_cache()

    # ---- the boundary collectives (TP > 1): NCCL bus bandwidth vs NVLink, share of the step
    comm_prof = None
    if world > 1 and not args.emulate_tp and strategy is Strategy.BOTTLENECK and args.boundary == "nccl":
        comm_prof = _comm_profile(args, pl, tp, world, dist, dev, ms)

    # ---- same-box baselines (north_star): the same kernels under naive low-rank TP and under
    # full-rank Megatron TP, same N, same block shape, same step (fwd+bwd+AdamW)
    baselines = None
    if not args.no_baselines and not args.model and strategy is Strategy.BOTTLENECK:
        baselines = {}
        for key, strat in (("naive_tp", Strategy.VANILLA), ("full_rank", Strategy.FULL_RANK)):
            if args.emulate_tp:
                from paper_2512_12131_b200.comm import TPComm

                comm = TPComm.emulated(tp, 0)
            tr, bpl, bvar, bx, bG = _make_trainer(args, cfg, strat, shape, comm)
            bxd, bgd = tr.device_inputs(bx, bG)
            bms, _ = _time_steps(args, tr, bxd, bgd, barrier)
            bms = _reduce_max(dist, world, bms, dev)
            lowrank = bvar is not Variant.FULL_RANK
            baselines[key] = {"value": b * s / (bms / 1e3), "unit": UNIT, "ms_per_step": bms,
                              "strategy": strat.value, "variant": bvar.value, "grouping": bpl.grouping,
                              "algorithmic_tflops_per_gpu": flops_per_step(cfg, b, s, lowrank=lowrank) / tp / (bms / 1e3) / 1e12}
            del tr, bxd, bgd
            if not args.dry_run:
                torch.cuda.empty_cache()
        baselines["btp_over_naive_tp"] = value / baselines["naive_tp"]["value"]
        baselines["btp_over_full_rank"] = value / baselines["full_rank"]["value"]
        baselines["targets"] = {"btp_over_naive_tp": 1.8, "btp_over_full_rank": 1.4, "at": "TP=8 (north_star)"}

    # ---- attention A/B at the step's attention shape (this rank's heads): our tcgen05 kernels vs the
    # cuDNN SDPA path the step uses, same process, CUDA events (evidence for profiles/attention)
    attention_ab = None
    if not args.dry_run and not args.no_attention_ab and not args.model and (world == 1 or args.share_gpu):
        attention_ab = _attention_ab(b, s, cfg.heads // tp, cfg.d // cfg.heads)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded uniform inputs, fan-in-scaled random init)",
        "config": {"workload": (f"CoLA-{args.config} model ({args.layers or cfg.layers} blocks + d-sharded embedding + "
                                f"replicated LM head V={args.vocab} + cross-entropy) " if args.model else
                                f"CoLA-{args.config} decoder block ")
                               + (f"[{variant.value} variant] " if variant not in (Variant.COLA, Variant.FULL_RANK)
                                  else "") + f"fwd+bwd{'' if args.no_optimizer else '+AdamW'}, "
                               f"{strategy.value} "
                               f"{'grouped ' if pl.grouping else ''}{'online-RMSNorm ' if pl.norm_mode.value == 'online' else ''}"
                               f"TP={tp}{' lowrank-ckpt' if pl.lowrank_ckpt else ''}",
                   "d": cfg.d, "d_ff": cfg.d_ff, "r": cfg.r, "heads": cfg.heads, "global_batch": b, "seq_len": s,
                   "tokens_per_step": b * s, "parallelism": f"tp{tp}", "l2": "inputs larger than L2 (no flush)",
                   "cuda_graph": graphed,
                   "boundary": args.boundary if tp > 1 else "none (tp=1)",
                   "boundary_dtype": args.boundary_dtype if tp > 1 else None,
                   "optimizer": None if args.no_optimizer else dict(ADAMW, kind="AdamW fp32 master+moments, fused"),
                   "attention": attention_label(args.attn, cfg, args)},
        "clocks": clk.summary() if clk is not None else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["dry-run"]},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roof,
        **({"roofline_attention_bwd": roof_att} if roof_att else {}),
        "algorithmic_tflops_per_gpu": flops / (ms / 1e3) / 1e12,
        "breakdown": breakdown,
    }
    if comm_prof is not None:
        line["comm"] = comm_prof
    if baselines is not None:
        line["baselines"] = baselines
    if attention_ab is not None:
        line["attention_ab"] = attention_ab
    if args.dry_run:
        line["dry_run"] = True
        line["data"] = "dry run (CPU, gloo): launch path and line schema only, NOT a measurement"
    if args.share_gpu:
        line["share_gpu"] = True
        line["data"] = "debug: all ranks on one GPU over gloo (N>1 code path only), NOT a measurement"
    if args.emulate_tp:
        line["metric"] = (f"EMULATED per-rank compute of a TP={tp} step on one GPU (collectives not executed; "
                          "value = tokens/s if comm were free; not the bench metric)")
        line["emulated_tp"] = tp
        line["scaling"] = None
        args.no_cpu_baseline = True
    if rank == 0 and not args.no_cpu_baseline:
        # the CPU arm runs on rank 0 only, after the timed work (other ranks wait at the barrier)
        rate, times, threads = cpu_oracle_rate(cfg, s, seconds_budget=args.cpu_seconds,
                                               max_steps=1 if args.dry_run else None)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"b=1 s={s} (1 of {b} sequences) CoLA-{args.config} block fwd+bwd, float64 "
                                          f"NumPy/BLAS oracle + AdamW, {len(times)} steps"}
        if not args.dry_run:
            line["cpu_baseline"]["reference_itself"] = _reference_itself()
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _self_launch(argv, gpus):
    """`python bench.py --gpus N` without torchrun: re-launch this script as N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1; rank 0's line is the output."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    # torchrun's own parser would take the short "--s" for an abbreviation of its options
    argv = ["--seq-len" if a == "--s" else "--batch" if a == "--b" else a for a in argv]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="1b")
    ap.add_argument("--b", "--batch", dest="b", type=int, default=4)
    ap.add_argument("--s", "--seq-len", dest="s", type=int, default=4096)
    ap.add_argument("--strategy", default="btp", choices=["btp", "vanilla", "full-rank"])
    ap.add_argument("--variant", default="cola", choices=["cola", "svd", "lax"],
                    help="low-rank block variant (lax: merges a resident seeded h bundle every step)")
    ap.add_argument("--ckpt", action="store_true")
    ap.add_argument("--no-grouping", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-optimizer", action="store_true", help="drop the AdamW update from the step")
    ap.add_argument("--no-fuse-sigma", action="store_true", help="TP=1: separate fix-up/sigma kernel (A/B)")
    ap.add_argument("--gemm-pair", type=int, default=-1, choices=[-1, 0, 1, 2],
                    help="CTA-pair GEMM tiles: 0 off, 1 plain/sigma epilogues, 2 also residual epilogues (A/B)")
    ap.add_argument("--gemm-st-global", type=int, default=-1, choices=[-1, 0, 1],
                    help="GEMM epilogue stores: 1 coalesced st.global, 0 TMA bulk stores (A/B)")
    ap.add_argument("--gemm-res", type=int, default=-1, choices=[-1, 0, 1, 2, 3],
                    help="residual-epilogue layout: 0 per-chunk, 1 whole tile, 2 producer-warp pipeline, "
                         "3 by width (default) (A/B)")
    ap.add_argument("--concurrent-wgrad", action="store_true", help="weight-gradient GEMMs on a side stream (A/B)")
    ap.add_argument("--no-merge-bwd-gemms", action="store_true",
                    help="launch each backward dgrad and its weight gradient separately (A/B)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-baselines", action="store_true", help="skip the naive-TP / full-rank same-box arms")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU + gloo: launch path, rendezvous and JSON schema only (contract test; no measurement)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--dump-gemms", default="", help="write per-launch GEMM timings (JSON) to this path")
    ap.add_argument("--attn", default="auto", choices=["auto", "cudnn", "flash", "native", "hybrid"])
    ap.add_argument("--attn-bwd-variant", type=int, default=-1, choices=[-1, 0, 1, 2],
                    help="hd-64 attention backward kernel (btp_attn_tune key 3): 0 shared warps, 1 split roles, "
                         "2 shared warps with the packed-P dS phase (A/B)")
    ap.add_argument("--no-attention-ab", action="store_true",
                    help="skip the in-process attention A/B (own kernels vs cuDNN) in the bench line")
    ap.add_argument("--share-gpu", action="store_true",
                    help="debug: all ranks on cuda:0 over gloo (exercises the N>1 path on one GPU; not a measurement)")
    ap.add_argument("--boundary", default="nccl", choices=["nccl", "peer", "nvls"],
                    help="TP>1 BTP chunk boundaries: NCCL all-reduce + fix-up, or the fused peer-memory kernels")
    ap.add_argument("--boundary-dtype", default="bf16", choices=["bf16", "fp32"],
                    help="NCCL boundaries: reduce the forward rank-r partials in fp32 (parity margin; 2x bytes)")
    ap.add_argument("--peer-provider", default="symmetric_memory", choices=["symmetric_memory", "cuda_ipc"],
                    help="--boundary peer/nvls: how the ranks' heaps are mapped")
    ap.add_argument("--model", action="store_true", help="multi-layer model step (embedding + blocks + LM head)")
    ap.add_argument("--layers", type=int, default=0, help="--model: number of blocks (default: the preset's)")
    ap.add_argument("--vocab", type=int, default=32000, help="--model: vocabulary size")
    ap.add_argument("--emulate-tp", type=int, default=0,
                    help="time ONE rank's compute of a TP=N plan on one GPU, collectives not executed "
                         "(compute-only; NOT the bench metric)")
    raw = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(raw, args.gpus)
    from paper_2512_12131_b200.model import COLA_60M, preset

    cfg = COLA_60M if args.config == "60m" else preset(args.config)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
