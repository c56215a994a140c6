"""CPU: the oracle's multi-layer model — analytic backward vs central finite
differences, and the package's model builder / token stream bit-equal to the oracle's."""

import numpy as np

from oracle import btp_oracle as O


import pytest


@pytest.mark.parametrize("variant,layers", [("cola", 2), ("lax", 3)])
def test_model_backward_matches_finite_differences(variant, layers):
    """lax: the h bundle chains the layers (h_cur of layer l is layer l+1's h_prev), so layer 0's
    down factors also receive gradient through every later layer's merge."""
    m = O.build_model(16, 40, 4, variant, 7, 24, layers)
    ids, tg = O.token_batch(2, 8, 24)
    loss, c = O.model_forward(m, ids, tg, 2, 8, 4)
    assert np.isfinite(loss) and 0 < loss < 10
    g = O.model_backward(m, c, 2, 8, 4)
    rng = np.random.default_rng(0)
    picks = [(lambda mm: mm["head"], g["dhead"]), (lambda mm: mm["embedding"], g["dembedding"]),
             (lambda mm: mm["final_gamma"], g["dfinal_gamma"]),
             (lambda mm: mm["blocks"][1]["A"]["q"], g["blocks"][1]["A"]["q"]),
             (lambda mm: mm["blocks"][0]["B"]["down"], g["blocks"][0]["B"]["down"]),
             (lambda mm: mm["blocks"][0]["gamma2"], g["blocks"][0]["dgamma2"])]
    for get, an in picks:
        P = get(m)
        for _ in range(3):
            idx = tuple(int(rng.integers(0, n)) for n in P.shape)
            if P is m["embedding"]:
                idx = (int(ids[rng.integers(0, len(ids))]),) + idx[1:]  # a row that is looked up
            h = 1e-6
            P[idx] += h
            lp, _ = O.model_forward(m, ids, tg, 2, 8, 4)
            P[idx] -= 2 * h
            lm, _ = O.model_forward(m, ids, tg, 2, 8, 4)
            P[idx] += h
            fd = (lp - lm) / (2 * h)
            assert abs(fd - an[idx]) <= 1e-6 * max(1.0, abs(fd)) + 1e-8, (idx, fd, an[idx])


def test_package_model_weights_and_tokens_equal_oracle():
    from paper_2512_12131_b200.model import ModelConfig, Variant, build_model, token_batch

    cfg = ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
    mw = build_model(cfg, Variant.COLA, 7, 24)
    om = O.build_model(16, 40, 4, "cola", 7, 24, 2)
    assert np.array_equal(mw.embedding.values, om["embedding"])
    assert np.array_equal(mw.head.values, om["head"])
    assert np.array_equal(mw.final_gamma.values, om["final_gamma"])
    for l in range(2):
        for n in O.PROJECTIONS:
            assert np.array_equal(mw.blocks[l].up_factors[n].values, om["blocks"][l]["A"][n])
            assert np.array_equal(mw.blocks[l].down_factors[n].values, om["blocks"][l]["B"][n])
    a, b = token_batch(3, 5, 24), O.token_batch(3, 5, 24)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[0].min() >= 0 and a[0].max() < 24
    assert np.array_equal(a[0].reshape(3, 5)[:, 1:], a[1].reshape(3, 5)[:, :-1])  # next-token targets
