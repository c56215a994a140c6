"""Device versions of the reference's tensor-level API (tensor.py:86-139, model.py:256-305):
matmul / batched_matmul / swiglu / reference_forward on host Tensors, against float64 NumPy and
the oracle block (fp32 mode: the north_star 1e-4 bar; the GEMM itself lands ~1e-7)."""

import numpy as np
import pytest

from oracle import btp_oracle as O
from paper_2512_12131_b200 import Tensor, batched_matmul, matmul, reference_forward, swiglu
from paper_2512_12131_b200.model import RunShape, Variant, build_block, fan_in_scaled, seeded_h_prev
from paper_2512_12131_b200.tensor import seeded_fill
from tests.gpu_util import SMALL, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n", [(37, 53, 29), (256, 512, 640), (1, 7, 3)])
def test_matmul_fp32_and_bf16(m, k, n):
    a, b = seeded_fill((m, k), 1), seeded_fill((k, n), 2)
    want = a.values @ b.values
    c, fl = matmul(a, b)
    assert fl == 2 * m * n * k and c.shape == (m, n)
    assert rel(c.values, want) < 1e-6
    c16, _ = matmul(a, b, precision="bf16")
    assert rel(c16.values, want) < 1e-2


def test_batched_matmul_is_bitwise_sequential():
    pairs = [(seeded_fill((64 + 8 * i, 40), 10 + i), seeded_fill((40, 24 + i), 20 + i)) for i in range(6)]
    outs, fl = batched_matmul(pairs)  # two grouped launches (4 + 2)
    assert fl == sum(2 * a.shape[0] * b.shape[1] * a.shape[1] for a, b in pairs)
    for (a, b), o in zip(pairs, outs):
        alone, _ = matmul(a, b)
        assert np.array_equal(o.values, alone.values)
        assert rel(o.values, a.values @ b.values) < 1e-6


def test_swiglu_matches_numpy():
    g, u = seeded_fill((3, 5, 7), 3), seeded_fill((3, 5, 7), 4)
    out = swiglu(g, u)
    assert out.shape == (3, 5, 7)
    assert rel(out.values, O.silu(g.values) * u.values) < 1e-6


@pytest.mark.parametrize("variant", ["cola", "svd", "lax", "full-rank"])
def test_reference_forward_vs_oracle(variant):
    b, s = 2, 64
    var = Variant(variant)
    blk = fan_in_scaled(build_block(SMALL, var, 0))
    oblk = O.build_block(SMALL.d, SMALL.d_ff, SMALL.r, variant, 0, scale_fan_in=3.0)
    x = seeded_fill((b, s, SMALL.d), 10000)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 1), 9) if var is Variant.LAX else None
    y, h = reference_forward(blk, x, hp)
    ohp = {n: t.values.reshape(b * s, -1) for n, t in hp.items()} if hp else None
    y_ref, c = O.block_forward(oblk, x.values.reshape(b * s, -1), b, s, SMALL.heads, h_prev=ohp)
    assert rel(y.values.reshape(b * s, -1), y_ref) < 1e-4
    if var is Variant.LAX:
        for n in O.PROJECTIONS:
            assert rel(h[n].values.reshape(b * s, -1), c["h_cur"][n]) < 1e-4
    else:
        assert h is None
