"""CPU: host-side scheduling decisions of the executor."""

import math

import pytest

from paper_2512_12131_b200.executor import _pick_splits, _pick_splits_behind


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


@pytest.mark.parametrize("tiles,kb", [(8, 256), (32, 256), (44, 256), (128, 256), (1, 8), (1000, 256)])
def test_split_k_picker_behind_nothing_equals_plain_picker(tiles, kb):
    """With no tiles ahead, the round-robin makespan model is the waves model of _pick_splits."""
    assert _pick_splits_behind([], tiles, kb, 74) == _pick_splits(tiles, kb, 74)


def test_split_k_picker_behind_a_dgrad_fills_its_last_wave():
    # o-chunk dgrad of the CoLA-1B step ([16384 x 512], K = 2048: 128 tiles of 32 k-blocks on 74 pairs,
    # the second wave 54 pairs deep) followed by its weight gradient [512 x 2048] over 256 k-blocks
    ahead = [32] * 128
    s = _pick_splits_behind(ahead, 8, 256, 74)
    loads = [0] * 74
    for j, c in enumerate(ahead + [-(-256 // s)] * (8 * s)):
        loads[j % 74] += c + 5
    # the merged launch is no longer than the two launches' models added
    alone = -(-128 // 74) * (32 + 5) + -(-8 * _pick_splits(8, 256, 74) // 74) * (-(-256 // _pick_splits(8, 256, 74)) + 5)
    assert max(loads) <= alone


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
