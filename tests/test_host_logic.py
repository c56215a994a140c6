"""CPU: host-side scheduling decisions of the executor."""

import math

import pytest

from paper_2512_12131_b200.executor import _pick_splits


@pytest.mark.parametrize("shapes,best", [
    # weight-gradient launches of the CoLA-1B step (T = 16384 tokens, 256 k-blocks); `best` is the
    # fastest split count of the measured B200 sweeps (tests/gpu_gemm_ab.py, tests/gpu_gemm_ab2.py)
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
