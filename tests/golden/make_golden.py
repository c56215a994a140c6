"""Generate golden vectors from the REFERENCE itself (btpsim, imported from /root/reference).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/btpsim_golden.npz + btpsim_golden.json. The files are committed; tests
read them, never the reference. Contents:

* seeded_fill known answers (several shapes/seeds)
* TOY config (reference test_simulator.py:24: d16 d_ff40 r4 h4, b2 s8, seed 7, x seed 8):
  y for every strategy x variant(svd, cola, full-rank) x tp{1,2,4} x online x grouping, the
  traced collective tuples, gemm launch counts, and every BTP per-rank workspace tensor
* SMALL config used by the GPU parity tests (d256 d_ff640 r64 h4, b2 s64, fan-in scaled
  weights): reference_forward y and the BTP tp=1 workspaces (online, grouped; float32)
* CoLA-60M block (b8 s256, fan-in scaled, cola): y checksums and per-intermediate norms
* `describe()` text for a set of plans
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import btpsim  # noqa: E402
from btpsim.model import (ModelConfig, RunShape, Variant, build_block, reference_forward,  # noqa: E402
                          seeded_h_prev)
from btpsim.plan import Strategy, describe, plan  # noqa: E402
from btpsim.simulator import execute_forward  # noqa: E402
from btpsim.tensor import Tensor, seeded_fill  # noqa: E402

OUT = Path(__file__).resolve().parent
TOY = ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
SMALL = ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)
C60M = ModelConfig(layers=8, heads=8, d=512, d_ff=1376, r=128)


def scaled(block):
    def sc(g):
        return {k: Tensor(v.values * np.sqrt(3.0 / v.shape[1]), v.element_bytes) for k, v in g.items()}

    return dataclasses.replace(block, full=sc(block.full), down_factors=sc(block.down_factors),
                               up_factors=sc(block.up_factors))


def main():
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"btpsim_version": btpsim.__version__, "combos": [], "describe": {}}

    for shape, seed in [((2, 3), 42), ((7,), 0), ((4, 5), 2**63 + 5), ((3, 3, 3), 123456789)]:
        key = f"fill_{'x'.join(map(str, shape))}_{seed}"
        arrays[key] = seeded_fill(shape, seed).values
        meta.setdefault("fills", []).append([list(shape), seed, key])

    # ---- TOY combos (mirrors reference test_simulator.py:47-55 `_run`)
    combos = [(Strategy.FULL_RANK, Variant.FULL_RANK), (Strategy.VANILLA, Variant.SVD),
              (Strategy.VANILLA, Variant.COLA), (Strategy.BOTTLENECK, Variant.SVD),
              (Strategy.BOTTLENECK, Variant.COLA)]
    for strategy, variant in combos:
        for tp in (1, 2, 4):
            if strategy is Strategy.VANILLA and (TOY.r % tp or (variant is Variant.COLA and (TOY.r // 2) % tp)):
                continue
            for online in (False, True):
                for grouping in (False, True):
                    shape = RunShape(b=2, s=8, tp=tp)
                    block = build_block(TOY, variant, seed=7)
                    x = seeded_fill((2, 8, TOY.d), 8)
                    v = None if strategy is Strategy.FULL_RANK else variant
                    pl = plan(strategy, TOY, shape, v, online_norm=online, grouping=grouping)
                    res = execute_forward(pl, block, x, model_tail=True)
                    tag = f"toy_{strategy.value}_{variant.value}_tp{tp}_on{int(online)}_g{int(grouping)}"
                    arrays[tag + "_y"] = res.y.values
                    entry = {"tag": tag, "strategy": strategy.value, "variant": variant.value, "tp": tp,
                             "online": online, "grouping": grouping,
                             "records": [list(map(lambda z: list(z) if isinstance(z, tuple) else z, r))
                                         for r in res.trace.record_tuples()],
                             "gemm_launches": res.trace.gemm_launches, "gemm_flops": res.trace.gemm_flops,
                             "ws_names": []}
                    if strategy is Strategy.BOTTLENECK:
                        for rk, ws in enumerate(res.workspaces):
                            for name, arr in ws.items():
                                arrays[f"{tag}_ws{rk}_{name}"] = np.asarray(arr)
                                if rk == 0:
                                    entry["ws_names"].append(name)
                    meta["combos"].append(entry)
    y_ref, _ = reference_forward(build_block(TOY, Variant.COLA, seed=7), seeded_fill((2, 8, TOY.d), 8))
    arrays["toy_cola_reference_y"] = y_ref.values

    # ---- TOY lax (cross-layer h bundle; reference test_acceptance.py:147-170): BTP with and
    # without a seeded h_prev (seed 9), y + the h_cur bundle + every per-rank workspace
    meta["lax"] = []
    for tp in (1, 2, 4):
        for online in (False, True):
            for grouping in (False, True):
                for hp_seed in (None, 9):
                    shape = RunShape(b=2, s=8, tp=tp)
                    block = build_block(TOY, Variant.LAX, seed=7)
                    x = seeded_fill((2, 8, TOY.d), 8)
                    hp = None if hp_seed is None else seeded_h_prev(TOY, shape, hp_seed)
                    pl = plan(Strategy.BOTTLENECK, TOY, shape, Variant.LAX, online_norm=online, grouping=grouping)
                    res = execute_forward(pl, block, x, hp, model_tail=True)
                    tag = f"toy_lax_tp{tp}_on{int(online)}_g{int(grouping)}_hp{hp_seed or 0}"
                    arrays[tag + "_y"] = res.y.values
                    for n, h in res.h_cur.items():
                        arrays[f"{tag}_h_{n}"] = h.values
                    names = []
                    for rk, ws in enumerate(res.workspaces):
                        for name, arr in ws.items():
                            arrays[f"{tag}_ws{rk}_{name}"] = np.asarray(arr)
                            if rk == 0:
                                names.append(name)
                    meta["lax"].append({"tag": tag, "tp": tp, "online": online, "grouping": grouping,
                                        "hp_seed": hp_seed, "ws_names": names,
                                        "records": [list(map(lambda z: list(z) if isinstance(z, tuple) else z, r))
                                                    for r in res.trace.record_tuples()]})
    yl, hl = reference_forward(build_block(TOY, Variant.LAX, seed=7), seeded_fill((2, 8, TOY.d), 8),
                               seeded_h_prev(TOY, RunShape(2, 8, 1), 9))
    arrays["toy_lax_reference_y"] = yl.values
    for n, h in hl.items():
        arrays[f"toy_lax_reference_h_{n}"] = h.values

    # ---- SMALL (GPU parity config), fan-in scaled
    blk = scaled(build_block(SMALL, Variant.COLA, seed=0))
    x = seeded_fill((2, 64, SMALL.d), 10000)
    arrays["small_cola_reference_y"] = reference_forward(blk, x)[0].values
    # float32 storage keeps the fixture small; it pins the oracle to ~1e-7 relative here, while
    # the TOY combos above pin it at float64 precision
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(2, 64, 1), Variant.COLA, online_norm=True, grouping=True)
    res = execute_forward(pl, blk, x)
    for name, arr in res.workspaces[0].items():
        arrays[f"small_tp1_ws0_{name}"] = np.asarray(arr, dtype=np.float32)
    meta["small"] = {"d": SMALL.d, "d_ff": SMALL.d_ff, "r": SMALL.r, "heads": SMALL.heads, "b": 2, "s": 64,
                     "seed": 0, "x_seed": 10000, "fan_in_gain": 3.0}

    # ---- CoLA-60M block checksums (reference forward ~10 s)
    blk60 = scaled(build_block(C60M, Variant.COLA, seed=0))
    x60 = seeded_fill((8, 256, C60M.d), 10000)
    pl60 = plan(Strategy.BOTTLENECK, C60M, RunShape(8, 256, 1), Variant.COLA, online_norm=True, grouping=True)
    res60 = execute_forward(pl60, blk60, x60)
    ws = res60.workspaces[0]
    meta["c60m"] = {
        "y_sum": float(res60.y.values.sum()),
        "y_head": res60.y.values.reshape(-1, C60M.d)[:2, :8].tolist(),
        "norms": {k: float(np.linalg.norm(v)) for k, v in ws.items()},
        "mlp_head": ws["mlp"][:2, :8].tolist(),
    }

    # ---- describe() goldens
    for strategy, variant, tp, online, grouping in [
        (Strategy.BOTTLENECK, Variant.COLA, 2, True, False),
        (Strategy.BOTTLENECK, Variant.COLA, 2, True, True),
        (Strategy.BOTTLENECK, Variant.SVD, 4, False, True),
        (Strategy.VANILLA, Variant.COLA, 2, True, True),
        (Strategy.VANILLA, Variant.LAX, 1, False, False),
        (Strategy.FULL_RANK, Variant.FULL_RANK, 4, False, True),
    ]:
        v = None if strategy is Strategy.FULL_RANK else variant
        pl = plan(strategy, TOY, RunShape(2, 8, tp), v, online_norm=online, grouping=grouping, lowrank_ckpt=True)
        meta["describe"][f"{strategy.value}|{variant.value}|{tp}|{int(online)}|{int(grouping)}"] = describe(pl)

    np.savez_compressed(OUT / "btpsim_golden.npz", **arrays)
    (OUT / "btpsim_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(f"{len(arrays)} arrays, {len(meta['combos'])} combos")


if __name__ == "__main__":
    main()
