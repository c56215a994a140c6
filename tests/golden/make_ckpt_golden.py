"""Reference CkptReport values at the GPU checkpoint test's configuration (SMALL d256 d_ff640
r64 h4, b2 s64, TP=2; reference checkpointing.py:109-163), generated from the REFERENCE itself.

    python tests/golden/make_ckpt_golden.py   # build container only; writes ckpt_small.json

The device's stored sets are what its backward reads (not the reference's workspace inventory),
so tests compare collective counts and ring elements exactly and ΔMem / eff_ckpt by ORDERING
(BTP vs naive TP) — which at this shape is the reference's own, not the TOY shape's of
reference test_ckpt.py:115-122 (at SMALL b2 s64 the reference itself ranks naive TP's svd eff
above BTP's)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from btpsim.checkpointing import CkptPolicy, run_with_ckpt  # noqa: E402
from btpsim.model import ModelConfig, RunShape, Variant, build_block, seeded_h_prev  # noqa: E402
from btpsim.plan import Strategy, plan  # noqa: E402
from btpsim.tensor import seeded_fill  # noqa: E402

SMALL = ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)


def main():
    b, s, tp = 2, 64, 2
    out = {}
    for strategy in ("btp", "vanilla"):
        for variant in ("svd", "lax", "cola"):
            for grouping in (True, False):
                var = Variant(variant)
                shape = RunShape(b, s, tp)
                blk = build_block(SMALL, var, 0)
                x = seeded_fill((b, s, SMALL.d), 10000)
                hp = seeded_h_prev(SMALL, shape, 5) if var is Variant.LAX else None
                pl = plan(Strategy(strategy), SMALL, shape, var, online_norm=strategy == "btp", grouping=grouping,
                          lowrank_ckpt=True)
                run = run_with_ckpt(pl, blk, x, CkptPolicy.LOWRANK_BOUNDARY, hp)
                out[f"{strategy}/{variant}/{int(grouping)}"] = run.report.to_dict()
    path = Path(__file__).resolve().parent / "ckpt_small.json"
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
