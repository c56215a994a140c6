"""Where does the bf16 parity error come from? (CPU, float64 simulation; not a test)

Re-runs the TP=1 block forward + backward of the oracle (oracle/btp_oracle.py, itself a restatement
of reference model.py:189-305) with a bf16 rounding applied at every point where the device path
stores a bf16 tensor, and switches each rounding point off in turn: the drop in the worst weight-
gradient error per point is that point's share of the error budget.

    python scripts/precision_budget.py [--cfg 60m] [--b 2 --s 128]
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import btp_oracle as O

POINTS = ("x", "w", "n", "z", "a", "proj", "attn", "xmid", "act", "dy", "da", "dP", "dh", "dgu", "dx", "dqkv")


def R(t, on):
    if not on:
        return t
    return torch.from_numpy(np.ascontiguousarray(t)).to(torch.bfloat16).double().numpy()


def run(blk0, x0, G0, b, s, heads, pts):
    r = lambda k, t: R(t, k in pts)  # noqa: E731
    blk = {"variant": "cola", "A": {n: r("w", v) for n, v in blk0["A"].items()},
           "B": {n: r("w", v) for n, v in blk0["B"].items()},
           "gamma1": r("w", blk0["gamma1"]), "gamma2": r("w", blk0["gamma2"])}
    x = r("x", x0)
    d = x.shape[1]
    hd = d // heads
    c = {}

    def proj(name, inp):
        z = r("z", inp @ blk["B"][name].T)
        a = r("a", O.crossgate(z))
        c["z_" + name], c["a_" + name] = z, a
        return a @ blk["A"][name].T

    n1 = r("n", O.rmsnorm(x, blk["gamma1"]))
    q, k, v = (r("proj", proj(nm, n1)) for nm in ("q", "k", "v"))
    attn, p = O.sdpa(q, k, v, b, s, heads, hd)
    attn = r("attn", attn)
    xm = r("xmid", x + proj("o", attn))
    n2 = r("n", O.rmsnorm(xm, blk["gamma2"]))
    gt, up = r("proj", proj("gate", n2)), r("proj", proj("up", n2))
    act = r("act", O.silu(gt) * up)
    y = r("xmid", xm + proj("down", act))
    dy = r("dy", G0)
    g = {"A": {}, "B": {}}

    def pbwd(name, inp, dout):
        g["A"][name] = dout.T @ c["a_" + name]
        da = r("da", dout @ blk["A"][name])
        dz = r("dP", O.crossgate_bwd(c["z_" + name], da))
        g["B"][name] = dz.T @ inp
        return dz @ blk["B"][name]

    dact = r("dh", pbwd("down", act, dy))
    dgate = r("dgu", dact * up * O.dsilu(gt))
    dup = r("dgu", dact * O.silu(gt))
    dn2 = r("dh", pbwd("gate", n2, dgate) + pbwd("up", n2, dup))
    dxm, g["g2"] = O._rmsnorm_bwd(xm, blk["gamma2"], dn2, O.EPS)
    dxm = r("dx", dxm + dy)
    dattn = r("dh", pbwd("o", attn, dxm))
    dq, dk, dv = (r("dqkv", t) for t in O.sdpa_bwd(dattn, q, k, v, p, b, s, heads, hd))
    dn1 = r("dh", pbwd("q", n1, dq) + pbwd("k", n1, dk) + pbwd("v", n1, dv))
    dx, g["g1"] = O._rmsnorm_bwd(x, blk["gamma1"], dn1, O.EPS)
    g["dx"] = dx + dxm
    g["y"] = y
    return g


def errs(g, ref):
    def rel(a, w):
        return float(np.linalg.norm(a - w) / np.linalg.norm(w))

    e = {"y": rel(g["y"], ref["y"]), "dx": rel(g["dx"], ref["dx"]), "g1": rel(g["g1"], ref["g1"]),
         "g2": rel(g["g2"], ref["g2"])}
    for fam in ("A", "B"):
        for n in O.PROJECTIONS:
            e[f"{fam}_{n}"] = rel(g[fam][n], ref[fam][n])
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--b", type=int, default=2)
    ap.add_argument("--s", type=int, default=128)
    args = ap.parse_args()
    d, d_ff, r, heads = 512, 1376, 128, 8
    blk = O.build_block(d, d_ff, r, "cola", 0, scale_fan_in=3.0)
    T = args.b * args.s
    x = O.seeded_fill((T, d), 10000)
    G = O.seeded_fill((T, d), 30000)
    ref = run(blk, x, G, args.b, args.s, heads, set())
    full = errs(run(blk, x, G, args.b, args.s, heads, set(POINTS)), ref)
    worst = max(full, key=full.get)
    print(f"all bf16 points: worst {worst} = {full[worst]:.3e}  (B_up {full['B_up']:.3e}, g2 {full['g2']:.3e})")
    for pt in POINTS:
        e = errs(run(blk, x, G, args.b, args.s, heads, set(POINTS) - {pt}), ref)
        w = max(e, key=e.get)
        print(f"  without {pt:5s}: worst {w:7s} = {e[w]:.3e}   B_up {e['B_up']:.3e}  g2 {e['g2']:.3e}")
    for pt in POINTS:
        e = errs(run(blk, x, G, args.b, args.s, heads, {pt}), ref)
        w = max(e, key=e.get)
        print(f"  only    {pt:5s}: worst {w:7s} = {e[w]:.3e}")


if __name__ == "__main__" and "--exact" not in sys.argv:
    main()


def inputs_exact():
    """The same budget when the inputs (x, weights) are bf16-exact, i.e. both sides get identical
    already-rounded inputs: what remains is the computation's own error."""
    d, d_ff, r, heads = 512, 1376, 128, 8
    blk = O.build_block(d, d_ff, r, "cola", 0, scale_fan_in=3.0)
    b, s = 2, 128
    x = O.seeded_fill((b * s, d), 10000)
    G = O.seeded_fill((b * s, d), 30000)
    pts = set(POINTS) - {"x", "w"}
    rb = {"variant": "cola", "A": {n: R(v, True) for n, v in blk["A"].items()},
          "B": {n: R(v, True) for n, v in blk["B"].items()}, "gamma1": R(blk["gamma1"], True),
          "gamma2": R(blk["gamma2"], True)}
    ref = run(rb, R(x, True), G, b, s, heads, set())
    e = errs(run(rb, R(x, True), G, b, s, heads, pts), ref)
    w = max(e, key=e.get)
    print(f"bf16-exact inputs: worst {w} = {e[w]:.3e}")


if __name__ == "__main__" and "--exact" in sys.argv:
    inputs_exact()
