"""BlockTrainer.fit (the bench's e2e path): the first batch's H2D goes out in row slices on several
copy streams, later batches on one stream under the previous step. The losses must equal those of
the same steps run one at a time through step() (single-stream copies)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("streams", [4, 1])
def test_fit_first_batch_sliced_copy_matches_step(streams):
    from tests.gpu_util import SMALL, inputs
    from paper_2512_12131_b200.api import BlockTrainer
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan

    b, s = 2, 128
    blk, x, G, _ = inputs(SMALL, Variant.COLA, b, s)
    x2 = x.values * 0.5 + 0.25  # a second, different batch
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    prev = BlockTrainer.FIRST_COPY_STREAMS
    BlockTrainer.FIRST_COPY_STREAMS = streams
    try:
        a = BlockTrainer(pl, blk, adamw=dict(lr=1e-3))
        xh, gh = a.pinned_host_inputs(x.values, G.values)
        xh2, _ = a.pinned_host_inputs(x2, G.values)
        got = a.fit([xh, xh2, xh, xh2], gh)
    finally:
        BlockTrainer.FIRST_COPY_STREAMS = prev
    ref_tr = BlockTrainer(pl, blk, adamw=dict(lr=1e-3))
    want = [ref_tr.step(h, gh) for h in (xh, xh2, xh, xh2)]
    torch.cuda.synchronize()
    # split-K weight gradients meet in an fp32 reduce-add of unfixed order: steps after the first
    # AdamW update may differ in the last bits
    assert got[0] == want[0]
    np.testing.assert_allclose(got, want, rtol=1e-4)
