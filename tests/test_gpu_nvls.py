"""NVLS (NVLink SHARP) form of the peer boundaries: btp_peer_boundary_{fwd,bwd}_nvls read the
owned rows through the heap's MULTICAST address (multimem.ld_reduce, fp32 accumulation in the
switch) and write a / dP / dss once with multimem.st (replicated to every member).

The box has one GPU, so the multicast object has one member (`LocalMulticastHeap`): the switch
"sum" is the identity and the replication has one target. That still runs every multimem
instruction for real, and against the pull kernels fed the same member plus all-zero peers the
results must be BIT-identical (the pull kernels also sum in fp32, and x + 0 is exact) — at a
tp=2/8 geometry too, which checks the owned-row indexing. Each case runs in a spawned process so a
faulting multimem instruction cannot take the test session's CUDA context with it.

A GPU that is not part of an NVLink multicast clique (e.g. a single GPU handed to a container: the
attribute CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED reads 1, but cuMulticastCreate returns
CUDA_ERROR_INVALID_VALUE) cannot create the object: the tests SKIP there, naming the error. The
NVLS kernels are the pull kernels' template instantiated with multicast load/store policies
(csrc/peer.cu), so the fix-up math they run is the one the pull tests pin."""

import ctypes

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _multicast_ok() -> bool:
    try:
        from cuda.bindings import driver as cu

        cu.cuInit(0)
        err, d0 = cu.cuDeviceGet(0)
        err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d0)
        return err == cu.CUresult.CUDA_SUCCESS and bool(v)
    except Exception:
        return False


def _kernels_main(tp, rank, variant, q):
    try:
        from paper_2512_12131_b200 import _native
        from paper_2512_12131_b200.peer import LocalMulticastHeap

        torch.manual_seed(7)
        dev, bf, f32 = "cuda:0", torch.bfloat16, torch.float32
        T, r, d = 512, 64, 256
        W = 3 * r
        own = T // tp
        # one multicast heap holding P | a | dA | dP | ss | dss (bf16 [T, W] x4, fp32 [T] x2)
        nb16, nb32 = T * W * 2, T * 4
        try:
            heap = LocalMulticastHeap(4 * nb16 + 2 * nb32, dev)
        except RuntimeError as e:
            q.put(({"skip": str(e)}, None))
            return
        H = heap.tensor
        offs = [0, nb16, 2 * nb16, 3 * nb16, 4 * nb16, 4 * nb16 + nb32]
        view = lambda i, dt, shp, nb: H[offs[i]:offs[i] + nb].view(dt).view(shp)  # noqa: E731
        P, A, dA, dP = (view(i, bf, (T, W), nb16) for i in range(4))
        ss, dss = view(4, f32, (T,), nb32), view(5, f32, (T,), nb32)
        H.zero_()
        P.copy_(torch.randn(T, W, device=dev))
        dA.copy_(torch.randn(T, W, device=dev))
        ss.copy_(torch.rand(T, device=dev) * d + 1.0)
        mc = lambda i: ctypes.c_void_p(heap.mc_ptr + offs[i])  # noqa: E731
        vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
        eps = ctypes.c_float(1e-6)

        # pull reference: peer 0 = the member's buffers, the other tp-1 "peers" contribute zeros
        zP, zS = torch.zeros(T, W, device=dev, dtype=bf), torch.zeros(T, device=dev, dtype=f32)
        refA = [torch.zeros(T, W, device=dev, dtype=bf) for _ in range(tp)]
        refdP = [torch.zeros(T, W, device=dev, dtype=bf) for _ in range(tp)]
        refdss = [torch.zeros(T, device=dev, dtype=f32) for _ in range(tp)]
        ptr = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)  # noqa: E731
        pP, pS = ptr([P] + [zP] * (tp - 1)), ptr([ss] + [zS] * (tp - 1))
        pdA = ptr([dA] + [zP] * (tp - 1))
        pA, pdP, pdss = ptr(refA), ptr(refdP), ptr(refdss)

        out = {}
        for form in ("pull", "nvls"):
            z_own = torch.zeros(own, W, device=dev, dtype=bf)
            s_own = torch.zeros(own, device=dev, dtype=f32)
            if form == "pull":
                rc = _native.call("btp_peer_boundary_fwd", vp(pP), vp(pS), tp, rank, T, W, r, variant, d, eps,
                                  vp(z_own), vp(s_own), vp(pA), st())
            else:
                rc = _native.call("btp_peer_boundary_fwd_nvls", mc(0), mc(4), tp, rank, T, W, r, variant, d, eps,
                                  vp(z_own), vp(s_own), mc(1), st())
            assert rc in (None, 0), rc
            if form == "pull":
                _native.call("btp_peer_boundary_bwd", vp(pdA), tp, rank, T, W, r, variant, d, vp(z_own), vp(s_own),
                             vp(pdP), vp(pdss), st())
            else:
                _native.call("btp_peer_boundary_bwd_nvls", mc(2), tp, rank, T, W, r, variant, d, vp(z_own),
                             vp(s_own), mc(3), mc(5), st())
            torch.cuda.synchronize()
            rows = slice(rank * own, (rank + 1) * own)
            if form == "pull":
                out[form] = (z_own.clone(), s_own.clone(), refA[0][rows].clone(), refdP[0][rows].clone(),
                             refdss[0][rows].clone())
            else:
                out[form] = (z_own.clone(), s_own.clone(), A[rows].clone(), dP[rows].clone(), dss[rows].clone())
        res = {}
        for i, nm in enumerate(("z", "s", "a", "dP", "dss")):
            x, y = out["pull"][i], out["nvls"][i]
            res[nm] = (bool(torch.equal(x, y)), float((x.float() - y.float()).abs().max()),
                       float(y.float().abs().max()))
        q.put((res, None))
    except BaseException:
        import traceback

        q.put((None, traceback.format_exc()))


def _step_main(variant, q):
    try:
        from tests.gpu_util import SMALL, inputs
        from paper_2512_12131_b200.api import make_executor, train_step
        from paper_2512_12131_b200.comm import TPComm
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.peer import PeerComm, VirtualPeers
        from paper_2512_12131_b200.plan import Strategy, plan
        from paper_2512_12131_b200.trace import Trace

        var = Variant(variant)
        b, s = 2, 64
        blk, x, G, _ = inputs(SMALL, var, b, s)
        pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), var, online_norm=True, grouping=True)
        got = {}
        for form in ("pull", "nvls"):
            provider = VirtualPeers(1) if form == "pull" else "local_multicast"
            pc = PeerComm(1, 0, "cuda:0", provider=provider)
            try:
                ex = make_executor(pl, blk, comm=TPComm(1, 0, trace=Trace(), peer=pc))
            except RuntimeError as e:
                if "multicast heap" not in str(e):
                    raise
                q.put(({"skip": str(e)}, None))
                return
            got[form] = train_step(pl, blk, x, G, executor=ex)
            torch.cuda.synchronize()
        a, n = got["pull"], got["nvls"]
        same = {"y": np.array_equal(a.y.values, n.y.values), "dx": np.array_equal(a.dx, n.dx),
                "loss": a.loss == n.loss}
        for fam in ("A", "B"):
            for k, g in a.grads[fam].items():
                same[f"d{fam}_{k}"] = np.array_equal(g, n.grads[fam][k])
        q.put((same, None))
    except BaseException:
        import traceback

        q.put((None, traceback.format_exc()))


def _spawn(target, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=target, args=(*args, q))
    p.start()
    try:
        res, err = q.get(timeout=600)
    finally:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert err is None, err
    if "skip" in res:
        pytest.skip(f"no multicast object on this GPU: {res['skip']}")
    return res


needs_mc = pytest.mark.skipif(not _multicast_ok(), reason="device reports no multicast (NVLS) support")


@needs_mc
@pytest.mark.parametrize("tp,rank", [(1, 0), (2, 1), (8, 5)])
@pytest.mark.parametrize("variant", [1, 0])
def test_nvls_kernels_match_pull(tp, rank, variant):
    res = _spawn(_kernels_main, tp, rank, variant)
    bad = {k: v for k, v in res.items() if not v[0]}
    assert not bad, bad
    assert res["a"][2] > 0 and res["dP"][2] > 0  # multimem stores landed


@needs_mc
@pytest.mark.parametrize("variant", ["cola", "svd"])
def test_nvls_step_bit_identical_to_pull(variant):
    same = _spawn(_step_main, variant)
    assert all(same.values()), same
