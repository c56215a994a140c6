"""Worst relative error (vs the float64 oracle) of the virtual-rank peer-boundary step, repeated:
python scripts/microbench/gpu_peer_margin.py TP SCATTER REPS  (not a pytest module)."""
import sys

sys.path.insert(0, ".")

if __name__ == "__main__":
    from tests.test_gpu_peer import _run_virtual
    from tests.gpu_util import SMALL, oracle_step, rel
    from oracle import btp_oracle as O

    tp, scatter, reps = int(sys.argv[1]), sys.argv[2] == "1", int(sys.argv[3])
    b, s = 2, 64
    for _ in range(reps):
        res, blk, x, G, oblk = _run_virtual(tp, SMALL, b, s, "cola", steps=2, scatter=scatter)
        y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=tp, sharded=False)
        dl = SMALL.d // tp
        errs = {"loss": abs(sum(v[1] for v in res.values()) - loss_ref) / abs(loss_ref)}
        for rank, (y, _, dx, grads, _, _) in res.items():
            gr = O.grads_for_rank(g_ref, tp, rank, SMALL.d, SMALL.d_ff)
            errs[f"y{rank}"] = rel(y, y_ref[:, rank * dl:(rank + 1) * dl])
            errs[f"dx{rank}"] = rel(dx, gr["dx"])
            for n in O.PROJECTIONS:
                errs[f"A_{n}{rank}"] = rel(grads["A"][n], gr["A"][n])
                errs[f"B_{n}{rank}"] = rel(grads["B"][n], gr["B"][n])
            errs[f"g1{rank}"] = rel(grads["gamma1"], gr["dgamma1"])
            errs[f"g2{rank}"] = rel(grads["gamma2"], gr["dgamma2"])
        w = max(errs, key=errs.get)
        print(f"tp={tp} scatter={scatter}: worst {w} = {errs[w]:.4e}", flush=True)
