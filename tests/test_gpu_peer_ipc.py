"""The peer-memory boundaries across real PROCESSES: tp rank processes share cuda:0 (time-sliced
contexts), each maps the others' heaps through CUDA IPC (`PeerComm(provider="cuda_ipc")`;
torch symmetric memory refuses several ranks on one device) and talks over a gloo group for
the host-side plumbing. Unlike the thread-based VirtualPeers tests, every rank has its own
address space and CUDA context, so the flags' system-scope release/acquire and the peer
mappings are exercised as on a multi-GPU node. Results against the float64 oracle per rank."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _rank_main(rank, world, port, scatter, variant, q):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=300))
        from tests.gpu_util import SMALL, inputs
        from paper_2512_12131_b200.api import make_executor, train_step
        from paper_2512_12131_b200.comm import TPComm
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.peer import PeerComm
        from paper_2512_12131_b200.plan import Strategy, plan
        from paper_2512_12131_b200.trace import Trace

        b, s = 2, 64
        var = Variant(variant)
        blk, x, G, _ = inputs(SMALL, var, b, s)
        pc = PeerComm(world, rank, "cuda:0", provider="cuda_ipc", scatter=scatter)
        comm = TPComm(world, rank, dist.group.WORLD, Trace(), peer=pc)
        pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, world), var, online_norm=True, grouping=True)
        ex = make_executor(pl, blk, comm=comm)
        for _ in range(2):  # the second step reuses the flags' epochs and every buffer
            st = train_step(pl, blk, x, G, executor=ex)
        torch.cuda.synchronize()
        q.put((rank, dict(y=st.y.values, loss=st.loss, dx=st.dx, grads=st.grads,
                          fwd=st.trace.record_tuples("forward")), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("world,scatter,variant", [(2, False, "cola"), (2, True, "cola"), (4, False, "cola"),
                                                   (2, False, "svd")])
def test_peer_boundaries_across_processes(world, scatter, variant):
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    env = {"CUDA_MODULE_LOADING": "EAGER"}  # no lazy module load behind a peer's spinning wait kernel
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        procs = [ctx.Process(target=_rank_main, args=(r, world, port, scatter, variant, q)) for r in range(world)]
        for p in procs:
            p.start()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    res = {}
    try:
        for _ in procs:
            rank, out, err = q.get(timeout=600)
            assert err is None, f"rank {rank} failed:\n{err}"
            res[rank] = out
    finally:
        for p in procs:
            p.join(timeout=60 if len(res) == world else 1)
            if p.is_alive():
                p.kill()
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant(variant), b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=world, sharded=False)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, world), Variant(variant), online_norm=True, grouping=True)
    pred = [(p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]
    for rank, o in res.items():
        assert rel(o["y"].reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(o["loss"] - loss_ref) / abs(loss_ref) < BF16_TOL
        gr = O.grads_for_rank(g_ref, world, rank, SMALL.d, SMALL.d_ff)
        errs = {"dx": rel(o["dx"], gr["dx"]), "gamma1": rel(o["grads"]["gamma1"], gr["dgamma1"]),
                "gamma2": rel(o["grads"]["gamma2"], gr["dgamma2"])}
        for n in O.PROJECTIONS:
            errs[f"A_{n}"] = rel(o["grads"]["A"][n], gr["A"][n])
            errs[f"B_{n}"] = rel(o["grads"]["B"][n], gr["B"][n])
        bad = {k: v for k, v in errs.items() if v > BF16_TOL}
        assert not bad, (rank, bad)
        assert o["fwd"][-len(pred):] == pred


def _model_rank_main(rank, world, port, q):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=300))
        from tests.test_gpu_model import B, S, _setup
        from paper_2512_12131_b200.comm import TPComm
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.model_executor import ModelExecutor, model_train_step
        from paper_2512_12131_b200.peer import PeerComm
        from paper_2512_12131_b200.plan import Strategy, plan
        from paper_2512_12131_b200.trace import Trace

        cfg, mw, ids, tg, _, _ = _setup()
        pl = plan(Strategy.BOTTLENECK, cfg, RunShape(B, S, world), Variant.COLA, online_norm=True, grouping=True)
        comm = TPComm(world, rank, dist.group.WORLD, Trace(), peer=PeerComm(world, rank, "cuda:0", provider="cuda_ipc"))
        ex = ModelExecutor(pl, mw, comm, "cuda:0")
        loss, ex = model_train_step(pl, mw, ids, tg, executor=ex)
        q.put((rank, dict(loss=loss, grads=ex.model_grads(), heaps=len({b.peer.heap.data_ptr() for b in ex.blocks})),
               None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, None, traceback.format_exc()))


def test_model_with_peer_boundaries_across_processes():
    """The multi-layer model over peer boundaries (one symmetric heap per block) at TP = 2."""
    from tests.test_gpu_model import _check_grads, _setup

    world = 2
    cfg, _, _, _, loss_ref, g_ref = _setup()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    os.environ["CUDA_MODULE_LOADING"] = "EAGER"
    try:
        procs = [ctx.Process(target=_model_rank_main, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
    finally:
        os.environ.pop("CUDA_MODULE_LOADING", None)
    res = {}
    try:
        for _ in procs:
            rank, out, err = q.get(timeout=600)
            assert err is None, f"rank {rank} failed:\n{err}"
            res[rank] = out
    finally:
        for p in procs:
            p.join(timeout=60 if len(res) == world else 1)
            if p.is_alive():
                p.kill()
    for rank, o in res.items():
        assert abs(o["loss"] - loss_ref) / abs(loss_ref) < 2e-2
        _check_grads(o["grads"], g_ref, tp=world, rank=rank, cfg=cfg)
        assert o["heaps"] == len(g_ref["blocks"])  # one peer heap per block
