"""Worst relative error per rank of the TP=4/8 C60M gloo runs vs the oracle (margin probe)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from tests import test_gpu_tp2 as T
from tests.gpu_util import C60M, inputs, oracle_step, rel
from oracle import btp_oracle as O
from paper_2512_12131_b200.model import Variant
def main():
    for world in (4, 8):
        b, s = 2, 128
        res = T._run_tp2("btp", True, True, False, world=world, cfg_name="C60M", bs=(b, s))
        blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
        y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, C60M, b, s, tp=world, online=True, sharded=False)
        worst = (0, None)
        for rank, (_, y, loss, dx, grads, *_r) in res.items():
            gr = O.grads_for_rank(g_ref, world, rank, C60M.d, C60M.d_ff)
            errs = {"y": rel(y.reshape(-1, C60M.d), y_ref), "dx": rel(dx, gr["dx"]), "g1": rel(grads["gamma1"], gr["dgamma1"]), "g2": rel(grads["gamma2"], gr["dgamma2"])}
            for n in O.PROJECTIONS:
                errs["A_" + n] = rel(grads["A"][n], gr["A"][n]); errs["B_" + n] = rel(grads["B"][n], gr["B"][n])
            k = max(errs, key=errs.get)
            if errs[k] > worst[0]: worst = (errs[k], (rank, k))
        print("world", world, "worst", worst)


if __name__ == "__main__":
    main()
