"""Which bf16 all-reduce drives the TP=4/8 worst error? Re-runs the C60M gloo TP step with the
boundary all-reduces done in fp32 (upcast -> reduce -> round once) for the forward, the backward,
both or neither, and prints the worst relative error per mode (experiment, GPU box)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.distributed as dist


def _patch(mode):
    from paper_2512_12131_b200 import comm as C

    def want(self):
        return mode == "both" or (mode == "fwd" and self.pass_tag != "backward") or (mode == "bwd" and self.pass_tag == "backward")

    def ar(self, buf):
        if buf.dtype == torch.bfloat16:
            f = buf.float()
            dist.all_reduce(f, group=self.group)
            buf.copy_(f)
        else:
            dist.all_reduce(buf, group=self.group)

    o_start, o_coal_start, o_coal, o_ar = (C.TPComm.all_reduce_start, C.TPComm.all_reduce_coalesced_start,
                                           C.TPComm.all_reduce_coalesced, C.TPComm.all_reduce)

    def all_reduce_start(self, buf, chunk_id, tag="block", record=True):
        if not want(self):
            return o_start(self, buf, chunk_id, tag, record)
        ar(self, buf)
        if record:
            self.trace.emit("all-reduce", chunk_id, tag, buf.numel(), self.pass_tag)
        return None

    def all_reduce_coalesced_start(self, main, stat, chunk_id, tag="block", stat_tag="fused-stat", record=True):
        if not want(self):
            return o_coal_start(self, main, stat, chunk_id, tag, stat_tag, record)
        ar(self, main); ar(self, stat)
        if record:
            self.trace.emit("all-reduce-coalesced", chunk_id, tag, main.numel(), self.pass_tag,
                            extras=((stat_tag, stat.numel()),))
        return None

    def all_reduce_coalesced(self, main, stat, chunk_id, tag="block", stat_tag="fused-stat"):
        if not want(self):
            return o_coal(self, main, stat, chunk_id, tag, stat_tag)
        ar(self, main); ar(self, stat)
        self.trace.emit("all-reduce-coalesced", chunk_id, tag, main.numel(), self.pass_tag,
                        extras=((stat_tag, stat.numel()),))
        return main, stat

    def all_reduce(self, buf, chunk_id, tag="block"):
        if not want(self):
            return o_ar(self, buf, chunk_id, tag)
        ar(self, buf)
        self.trace.emit("all-reduce", chunk_id, tag, buf.numel(), self.pass_tag)
        return buf

    C.TPComm.all_reduce_start = all_reduce_start
    C.TPComm.all_reduce_coalesced_start = all_reduce_coalesced_start
    C.TPComm.all_reduce_coalesced = all_reduce_coalesced
    C.TPComm.all_reduce = all_reduce


def rank_main(mode, *args):
    _patch(mode)
    from tests import test_gpu_tp2 as T
    T._rank_main(*args)


def run(mode, world, b, s, cfg_name="C60M"):
    import torch.multiprocessing as mp
    from tests import test_gpu_tp2 as T

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = T._port()
    procs = [ctx.Process(target=rank_main, args=(mode, r, world, port, "btp", True, True, False, q, cfg_name, (b, s)))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        item = q.get(timeout=600)
        assert item[-1] is None, item[-1]
        res[item[0]] = item
    for p in procs:
        p.join()
    return res


def main():
    import argparse

    from oracle import btp_oracle as O
    from tests import gpu_util
    from tests.gpu_util import inputs, oracle_step, rel
    from paper_2512_12131_b200.model import Variant

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C60M")
    ap.add_argument("--bs", default="2,128")
    ap.add_argument("--worlds", default="1,8")
    ap.add_argument("--modes", default="none,fwd,bwd,both")
    a = ap.parse_args()
    cfg = getattr(gpu_util, a.cfg)
    b, s = (int(v) for v in a.bs.split(","))
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    y_ref, g_ref, _, _ = oracle_step(oblk, x, G, cfg, b, s, sharded=False)
    for world in (int(w) for w in a.worlds.split(",")):
        for mode in (("none",) if world == 1 else a.modes.split(",")):
            res = run(mode, world, b, s, a.cfg)
            worst = {}
            for rank, (_, y, loss, dx, grads, *_r) in res.items():
                gr = O.grads_for_rank(g_ref, world, rank, cfg.d, cfg.d_ff)
                errs = {"y": rel(y.reshape(-1, cfg.d), y_ref), "dx": rel(dx, gr["dx"]),
                        "g1": rel(grads["gamma1"], gr["dgamma1"]), "g2": rel(grads["gamma2"], gr["dgamma2"])}
                for n in O.PROJECTIONS:
                    errs["A_" + n] = rel(grads["A"][n], gr["A"][n])
                    errs["B_" + n] = rel(grads["B"][n], gr["B"][n])
                for k, v in errs.items():
                    worst[k] = max(worst.get(k, 0), v)
            top = sorted(worst.items(), key=lambda kv: -kv[1])[:5]
            print(f"{a.cfg} b{b} s{s} world={world} mode={mode}: " + ", ".join(f"{k}={v:.3e}" for k, v in top),
                  flush=True)


if __name__ == "__main__":
    main()
