"""CPU: host-side scheduling decisions of the executor."""

import math

import pytest

from paper_2512_12131_b200.executor import _pick_splits


@pytest.mark.parametrize("shapes,best", [
    # weight-gradient launches of the CoLA-1B step (T = 16384 tokens, 256 k-blocks); `best` is the
    # fastest split count of the measured B200 sweeps (scripts/microbench/gpu_gemm_ab.py, scripts/microbench/gpu_gemm_ab2.py)
    ([(1024, 2048)], 2),
    ([(512, 2048)], 9),
    ([(5472, 512)], 5),
    ([(512, 5472)], 5),
    ([(5472, 512)] * 2, 5),
    ([(2048, 512)] * 3, 3),
    ([(1536, 2048)], 3),
])
def test_split_k_picker_matches_measured_optimum(shapes, best):
    tiles = sum(math.ceil(m / 256) * math.ceil(n / 256) for m, n in shapes)
    assert _pick_splits(tiles, 256, 74) == best


def test_split_k_picker_limits():
    assert _pick_splits(1000, 256, 74) == 1        # plenty of tiles: no split
    assert _pick_splits(1, 8, 74) == 2             # >= 4 k-blocks per split
    assert _pick_splits(1, 2, 74) == 1


def test_tensor_ops_errors_match_reference():
    """Shape errors of the device tensor ops are raised before any device work (tensor.py:86-139)."""
    import pytest as _pt

    from paper_2512_12131_b200 import batched_matmul, matmul, reference_forward, swiglu
    from paper_2512_12131_b200.model import ModelConfig, Variant, build_block
    from paper_2512_12131_b200.tensor import DimensionError, seeded_fill

    with _pt.raises(DimensionError, match="2-D"):
        matmul(seeded_fill((2, 3, 4), 0), seeded_fill((4, 2), 0))
    with _pt.raises(DimensionError, match="inner dimensions"):
        matmul(seeded_fill((2, 3), 0), seeded_fill((4, 2), 0))
    with _pt.raises(DimensionError, match="at least one"):
        batched_matmul([])
    with _pt.raises(DimensionError, match="disagree"):
        swiglu(seeded_fill((2, 3), 0), seeded_fill((3, 2), 0))
    blk = build_block(ModelConfig(layers=1, heads=4, d=16, d_ff=40, r=4), Variant.COLA, 0)
    with _pt.raises(DimensionError):
        reference_forward(blk, seeded_fill((2, 8, 15), 0))
