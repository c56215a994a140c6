"""CPU: bench.py's reference arm prints one JSON line with the driver's contract keys (the GPU arm
is exercised on the box)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "60m", "--b", "1",
                          "--s", "64", "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus2_self_launch_dry_run_json_line():
    """`bench.py --gpus 2` without torchrun re-launches itself as two ranks (torch.distributed.run,
    127.0.0.1); --dry-run swaps the device work for a CPU stand-in over gloo, so the launch path,
    barriers, max-over-ranks reductions, the boundary-collective profile, the same-box baselines
    and the rank-0 JSON line are exercised here without a GPU."""
    import os

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--config", "60m",
                          "--b", "1", "--s", "64", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline",
                "cpu_baseline", "baselines", "comm"):
        assert key in d, key
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3 and d["dry_run"] is True
    assert d["config"]["parallelism"] == "tp2"
    for key in ("h2d_bytes_per_step", "d2h_bytes_per_step", "value", "unit"):
        assert key in d["e2e"], key
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in d["roofline"], key
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    bl = d["baselines"]
    assert bl["naive_tp"]["strategy"] == "vanilla" and bl["full_rank"]["strategy"] == "full-rank"
    assert bl["btp_over_naive_tp"] > 0 and bl["btp_over_full_rank"] > 0
    cm = d["comm"]
    assert cm["backend"] == "gloo" and len(cm["per_boundary_fwd"]) == 4  # grouped BTP: 4 chunk boundaries
    assert all(r["bus_gbs"] > 0 for r in cm["per_boundary_fwd"]) and cm["peak_gbs"] == 900.0
