"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports btpsim; this test never does)."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import btp_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
ARR = np.load(GOLD / "btpsim_golden.npz")
META = json.loads((GOLD / "btpsim_golden.json").read_text())
TOY = dict(d=16, d_ff=40, r=4, heads=4, b=2, s=8)


def test_seeded_fill_known_answers():
    for shape, seed, key in META["fills"]:
        assert np.array_equal(O.seeded_fill(tuple(shape), seed), ARR[key]), key
    # KAT quoted in SURVEY §8c
    assert O.seeded_fill((2, 3), 42)[0, 0] == 0.4831297575436466


def test_reference_forward_toy_cola():
    blk = O.build_block(16, 40, 4, "cola", 7)
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y, _ = O.block_forward(blk, x, 2, 8, 4)
    np.testing.assert_allclose(y, ARR["toy_cola_reference_y"].reshape(16, 16), rtol=0, atol=1e-10)


@pytest.mark.parametrize("entry", [e for e in META["combos"]], ids=lambda e: e["tag"])
def test_toy_combo_outputs(entry):
    """Every strategy/variant/tp/online/grouping combo: the single-device oracle reproduces the
    reference's sharded y (the reference asserts the same equivalence at 1e-9)."""
    var = entry["variant"]
    blk = O.build_block(16, 40, 4, var, 7)
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y, _ = O.block_forward(blk, x, 2, 8, 4)
    np.testing.assert_allclose(y, ARR[entry["tag"] + "_y"].reshape(16, 16), rtol=0, atol=1e-9)


BTP = [e for e in META["combos"] if e["strategy"] == "btp"]


@pytest.mark.parametrize("entry", BTP, ids=lambda e: e["tag"])
def test_btp_sharded_workspaces(entry):
    """Per-rank, per-intermediate equality of the oracle's sharded BTP forward with the
    reference simulator's workspaces (incl. the online norm's locally normalised n1/n2)."""
    var, tp, online = entry["variant"], entry["tp"], entry["online"]
    blk = O.build_block(16, 40, 4, var, 7)
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y, ws = O.btp_forward_sharded(blk, x, 2, 8, 4, tp, online=online)
    np.testing.assert_allclose(y, ARR[entry["tag"] + "_y"].reshape(16, 16), rtol=0, atol=1e-9)
    for rk in range(tp):
        for name in entry["ws_names"]:
            want = ARR[f"{entry['tag']}_ws{rk}_{name}"]
            got = ws[rk][name]
            np.testing.assert_allclose(np.asarray(got).reshape(want.shape), want, rtol=1e-9, atol=1e-9,
                                       err_msg=f"rank {rk} {name}")


def test_small_config_workspaces():
    m = META["small"]
    blk = O.build_block(m["d"], m["d_ff"], m["r"], "cola", m["seed"], scale_fan_in=m["fan_in_gain"])
    x = O.seeded_fill((m["b"], m["s"], m["d"]), m["x_seed"]).reshape(-1, m["d"])
    y, c = O.block_forward(blk, x, m["b"], m["s"], m["heads"])
    np.testing.assert_allclose(y, ARR["small_cola_reference_y"].reshape(y.shape), rtol=0, atol=1e-10)
    _, ws = O.btp_forward_sharded(blk, x, m["b"], m["s"], m["heads"], 1, online=True)
    for name in ws[0]:
        want = ARR[f"small_tp1_ws0_{name}"]
        got = np.asarray(ws[0][name], dtype=np.float64).reshape(want.shape)
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err < 1e-6, (name, err)


def test_c60m_checksums():
    m = META["c60m"]
    blk = O.build_block(512, 1376, 128, "cola", 0, scale_fan_in=3.0)
    x = O.seeded_fill((8, 256, 512), 10000).reshape(-1, 512)
    y, ws = O.btp_forward_sharded(blk, x, 8, 256, 8, 1, online=True)
    assert abs(y.sum() - m["y_sum"]) <= 1e-9 * max(1.0, abs(m["y_sum"])) * 100
    np.testing.assert_allclose(y[:2, :8], np.array(m["y_head"]), rtol=0, atol=1e-10)
    np.testing.assert_allclose(ws[0]["mlp"][:2, :8], np.array(m["mlp_head"]), rtol=1e-9, atol=1e-12)
    for name, nrm in m["norms"].items():
        got = np.linalg.norm(np.asarray(ws[0][name]))
        assert abs(got - nrm) <= 1e-9 * nrm, name


def _toy_hp(seed):
    if seed is None:
        return None
    return {n: h.reshape(16, 4) for n, h in O.seeded_h_prev(2, 8, 4, seed).items()}


def test_reference_forward_toy_lax():
    """reference_forward with a seeded h bundle (model.py:256-305): y and the returned h_cur."""
    blk = O.build_block(16, 40, 4, "lax", 7)
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y, c = O.block_forward(blk, x, 2, 8, 4, h_prev=_toy_hp(9))
    np.testing.assert_allclose(y, ARR["toy_lax_reference_y"].reshape(16, 16), rtol=0, atol=1e-10)
    for n in O.PROJECTIONS:
        np.testing.assert_allclose(c["h_cur"][n], ARR[f"toy_lax_reference_h_{n}"].reshape(16, 4), rtol=0, atol=1e-12)


def test_lax_without_h_prev_is_svd():
    """reference test_model.py:182-192: LaX with no (zero) bundle equals SVD."""
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y_svd, _ = O.block_forward(O.build_block(16, 40, 4, "svd", 7), x, 2, 8, 4)
    y_lax, _ = O.block_forward(O.build_block(16, 40, 4, "lax", 7), x, 2, 8, 4)
    y_zero, _ = O.block_forward(O.build_block(16, 40, 4, "lax", 7), x, 2, 8, 4,
                                h_prev={n: np.zeros((16, 4)) for n in O.PROJECTIONS})
    assert np.array_equal(y_svd, y_lax) and np.array_equal(y_svd, y_zero)


@pytest.mark.parametrize("entry", META["lax"], ids=lambda e: e["tag"])
def test_btp_lax_sharded_workspaces(entry):
    """BTP lax under every tp/online/grouping, with and without an h bundle: y, the h_cur bundle
    (= the replicated z) and every per-rank workspace of the reference simulator."""
    tp, online = entry["tp"], entry["online"]
    blk = O.build_block(16, 40, 4, "lax", 7)
    x = O.seeded_fill((2, 8, 16), 8).reshape(16, 16)
    y, ws = O.btp_forward_sharded(blk, x, 2, 8, 4, tp, online=online, h_prev=_toy_hp(entry["hp_seed"]))
    np.testing.assert_allclose(y, ARR[entry["tag"] + "_y"].reshape(16, 16), rtol=0, atol=1e-9)
    for n in O.PROJECTIONS:
        np.testing.assert_allclose(ws[0][f"z_{n}"], ARR[f"{entry['tag']}_h_{n}"].reshape(16, 4), rtol=1e-9,
                                   atol=1e-9)
    for rk in range(tp):
        assert set(entry["ws_names"]) == set(ws[rk]), set(entry["ws_names"]) ^ set(ws[rk])
        for name in entry["ws_names"]:
            want = ARR[f"{entry['tag']}_ws{rk}_{name}"]
            np.testing.assert_allclose(np.asarray(ws[rk][name]).reshape(want.shape), want, rtol=1e-9, atol=1e-9,
                                       err_msg=f"rank {rk} {name}")
