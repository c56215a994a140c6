"""Probe: does torch symmetric memory give a multicast (NVLS) address on this box (1 rank)?"""
import datetime
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29655")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, timeout=datetime.timedelta(seconds=60),
                        device_id=torch.device("cuda", 0))
dev = torch.cuda.current_device()
from cuda.bindings import driver as cu
cu.cuInit(0)
err, d0 = cu.cuDeviceGet(0)
err, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d0)
print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", err, mc)
t = symm_mem.empty(1 << 20, dtype=torch.uint8, device="cuda")
hdl = symm_mem.rendezvous(t, dist.group.WORLD)
print("backend", symm_mem.get_backend("cuda") if hasattr(symm_mem, "get_backend") else "?")
from torch._C._distributed_c10d import _SymmetricMemory
print("has_multicast_support", _SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, 0)
      if hasattr(torch._C, "_autograd") else "?", "multicast_ptr", hdl.multicast_ptr)
dist.destroy_process_group()
