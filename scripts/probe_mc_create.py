"""Probe: which cuMulticastCreate property sets does this box accept (one-device objects)?"""
import torch
from cuda.bindings import driver as cu

torch.empty(1, device="cuda")
H = cu.CUmemAllocationHandleType
for ht in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    for nd in (1, 2):
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = nd
        mp.handleTypes = getattr(H, ht)
        mp.size = 2 << 20
        g = cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        g2 = cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        if g[0] == cu.CUresult.CUDA_SUCCESS:
            mp.size = max(g[1], 2 << 20)
        r = cu.cuMulticastCreate(mp)
        print(ht, nd, "gran", g, g2, "create", r[0])
