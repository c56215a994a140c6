"""Multi-process (world_size 2, gloo, CPU) coverage of the TP communicator: in-place sums,
the coalesced rider record, the d-axis gather, and record schema/pass tags."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_12131_b200.comm import TPComm
from paper_2512_12131_b200.trace import Trace, ring_transfer_elements, trace_volume


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TPComm.from_env(world, trace=Trace())
        main = torch.full((4, 3), float(rank + 1), dtype=torch.bfloat16)
        stat = torch.full((4,), 10.0 * (rank + 1))
        comm.all_reduce_coalesced(main, stat, "qkv")
        part = torch.full((4, 2), float(rank))
        comm.all_reduce(part, "o")
        comm.pass_tag = "backward"
        comm.all_reduce(torch.ones(4, 2), "o")
        shard = torch.arange(8, dtype=torch.float32).view(4, 2) + 100 * rank
        comm.pass_tag = "forward"
        full = comm.all_gather_cols(shard, "final-gather")
        q.put((rank, main.float().tolist(), stat.tolist(), part.tolist(), full.tolist(),
               comm.trace.record_tuples(), trace_volume(comm.trace, tag="block", pass_tag="forward"),
               ring_transfer_elements(comm.trace, world, pass_tag="forward")))
    finally:
        dist.destroy_process_group()


def test_tp2_collectives_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, main, stat, part, full, recs, vol, ring in out:
        assert main == [[3.0] * 3] * 4
        assert stat == [30.0] * 4
        assert part == [[1.0] * 2] * 4
        assert full[0] == [0.0, 1.0, 100.0, 101.0]
        assert recs == [
            ("qkv", "all-reduce-coalesced", "block", 12, (("fused-stat", 4),)),
            ("o", "all-reduce", "block", 8, ()),
            ("o", "all-reduce", "block", 8, ()),
            ("final-gather", "all-gather", "boundary", 16, ()),
        ]
        assert vol == (20, 40, 2)
        assert ring == 2 * (12 + 4 + 8 + 16)


def test_single_rank_still_records():
    comm = TPComm(1, 0)
    buf = torch.ones(2, 2)
    comm.all_reduce(buf, "solo")
    assert comm.trace.record_tuples() == [("solo", "all-reduce", "block", 4, ())]
    assert torch.equal(buf, torch.ones(2, 2))


def test_emulated_comm_records_without_exchange():
    """TPComm.emulated: one rank's share of a tp-way plan on one device, no process group; every
    collective is recorded with the reference schema but nothing is exchanged."""
    comm = TPComm.emulated(8, 3)
    assert comm.tp == 8 and comm.rank == 3 and not comm.live
    buf = torch.full((4, 2), 2.0)
    comm.all_reduce(buf, "o")
    comm.all_reduce_coalesced(buf, torch.ones(4), "qkv")
    assert comm.wait(comm.all_reduce_start(buf, "down")) is None
    assert torch.equal(buf, torch.full((4, 2), 2.0))
    assert comm.all_gather_cols(torch.ones(4, 2), "final-gather").shape == (4, 16)
    assert [r[0] for r in comm.trace.record_tuples()] == ["o", "qkv", "down", "final-gather"]
    with pytest.raises(ValueError):
        TPComm.emulated(2, 2)
