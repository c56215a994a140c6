"""Probe: a peer heap (cuda_ipc, or torch symmetric memory) across TWO processes sharing cuda:0 (gloo group),
then a device-side signal/wait exchange through libbtp's peer flags (time-sliced contexts)."""
import datetime
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, ".")


def main(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        from paper_2512_12131_b200.peer import PeerComm, READY

        pc = PeerComm(world, rank, "cuda:0", provider=sys.argv[1] if len(sys.argv) > 1 else "cuda_ipc")
        pc.setup([("buf", (1024,), torch.float32)])
        print(rank, "bases", [hex(b) for b in pc.bases], flush=True)
        for i in range(3):
            pc.exchange(READY)
            torch.cuda.synchronize()
        print(rank, "exchange ok", flush=True)
    except Exception as e:
        print(rank, "FAILED", type(e).__name__, str(e)[:300], flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(main, args=(2, 29611), nprocs=2)
