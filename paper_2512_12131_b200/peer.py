"""Symmetric peer-memory heap + signal flags for the fused BTP chunk boundaries (csrc/peer.cu).

Every rank carves the SAME list of buffers at the SAME offsets out of one heap allocation, so a
buffer's address on rank j is `base_j + offset`. The boundary kernels receive, per buffer, a
device array of the tp addresses (rank order) and pull/push rows over NVLink.

Two providers of the per-rank heap bases:

* `symmetric_memory` (the box): `torch.distributed._symmetric_memory.empty` + `rendezvous`
  over the job's process group — cuMem allocations exported to and mapped by every peer GPU.
  PyTorch is only plumbing here: the kernels that move and reduce the data are libbtp's.
* `VirtualPeers` (tests): tp ranks as tp threads of ONE process on ONE GPU, each with its own
  CUDA stream; the "peer" buffers are plain device allocations of the same GPU. The kernels,
  flags and executor code are exactly those of the multi-GPU path, so the single-GPU box can
  check the multi-rank numerics and the signal/wait protocol.
* `"cuda_ipc"`: a plain cudaMalloc heap per rank, exported with cudaIpcGetMemHandle and mapped by
  every other rank (handles exchanged over the process group) — the same heap without torch's
  symmetric-memory allocator. CUDA IPC also maps between processes on ONE device (where
  symmetric memory refuses), so the single-GPU box runs the real multi-process protocol: tp rank
  processes, time-sliced contexts, system-scope flags across address spaces.
* `"local_multicast"` (tests, tp=1): the heap is a cuMem allocation bound to a ONE-device NVSwitch
  multicast object (`LocalMulticastHeap`), so the NVLS kernels' multimem instructions run for real
  on a single-GPU box (the switch "sum" over one member is the identity).

nvls=True additionally gives every buffer a MULTICAST address (symmetric memory's multicast_ptr, or
the local multicast object) and the boundaries run as btp_peer_boundary_{fwd,bwd}_nvls: the switch
reduces the partials (multimem.ld_reduce) and replicates a / dP (multimem.st).
"""

from __future__ import annotations

import ctypes
import threading

import torch

from . import _native

READY, DONE = 0, 1   # flag slots: "my partial is written" / "my pushes have landed"
N_SLOTS = 2
_ALIGN = 256


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class VirtualPeers:
    """Registry shared by the tp threads of a single-GPU multi-rank run."""

    def __init__(self, tp: int):
        self.tp = tp
        self.bases = [0] * tp
        self._barrier = threading.Barrier(tp, timeout=300)  # a dead rank breaks the barrier, not the test

    def exchange(self, rank: int, base: int) -> list[int]:
        self.bases[rank] = base
        self._barrier.wait()
        out = list(self.bases)
        self._barrier.wait()  # nobody re-registers before everyone has read
        return out

    def barrier(self):
        self._barrier.wait()


class LocalMulticastHeap:
    """`nbytes` of device memory mapped twice: at a unicast address (wrapped as a torch uint8 tensor)
    and at the address of a one-device multicast object it is bound to (cuMulticastCreate /
    AddDevice / BindMem + cuMemMap). Single-GPU stand-in for symmetric memory's multicast mapping."""

    def __init__(self, nbytes: int, device):
        from cuda.bindings import driver as cu

        self._cu = cu
        dev = torch.device(device)
        torch.cuda.init()
        torch.empty(1, device=dev)  # primary context current on this thread

        def ok(res):
            err, *rest = res if isinstance(res, tuple) else (res,)
            if err != cu.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"multicast heap: {err}")
            return rest[0] if len(rest) == 1 else rest

        ordinal = dev.index if dev.index is not None else torch.cuda.current_device()
        cudev = ok(cu.cuDeviceGet(ordinal))
        if not ok(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev)):
            raise RuntimeError("device has no multicast (NVLS) support")
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mp.size = max(int(nbytes), 1)
        gran = ok(cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = -(-max(int(nbytes), 1) // gran) * gran
        mp.size = size
        self.mc_handle = ok(cu.cuMulticastCreate(mp))
        ok(cu.cuMulticastAddDevice(self.mc_handle, cudev))
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = ordinal
        ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.mem = ok(cu.cuMemCreate(size, ap, 0))
        ok(cu.cuMulticastBindMem(self.mc_handle, 0, self.mem, 0, size, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = ordinal
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = ok(cu.cuMemAddressReserve(size, gran, 0, 0))
        ok(cu.cuMemMap(self.uc, size, 0, self.mem, 0))
        ok(cu.cuMemSetAccess(self.uc, size, [acc], 1))
        self.mc = ok(cu.cuMemAddressReserve(size, gran, 0, 0))
        ok(cu.cuMemMap(self.mc, size, 0, self.mc_handle, 0))
        ok(cu.cuMemSetAccess(self.mc, size, [acc], 1))
        self.size = size
        self.uc_ptr, self.mc_ptr = int(self.uc), int(self.mc)
        holder = type("_UC", (), {})()
        holder.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                           "data": (self.uc_ptr, False), "version": 3}
        self.tensor = torch.as_tensor(holder, device=dev)
        self._holder = holder


class IpcHeap:
    """`nbytes` of cudaMalloc'd device memory (a whole allocation, so an IPC handle maps its base),
    wrapped as a torch uint8 tensor, plus the mapped bases of other ranks' heaps."""

    def __init__(self, nbytes: int, device):
        from cuda.bindings import runtime as rt

        self._rt = rt
        dev = torch.device(device)
        torch.empty(1, device=dev)  # context current
        err, ptr = rt.cudaMalloc(max(int(nbytes), 1))
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"ipc heap: cudaMalloc {err}")
        self.ptr = int(ptr)
        holder = type("_IPC", (), {})()
        holder.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (self.ptr, False),
                                           "version": 3}
        self.tensor = torch.as_tensor(holder, device=dev)
        self._holder = holder
        self._opened: list[int] = []

    def handle(self) -> bytes:
        err, h = self._rt.cudaIpcGetMemHandle(self.ptr)
        if err != self._rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"ipc heap: cudaIpcGetMemHandle {err}")
        return bytes(h.reserved)

    def open(self, handle: bytes) -> int:
        h = self._rt.cudaIpcMemHandle_t()
        h.reserved = list(handle)
        err, ptr = self._rt.cudaIpcOpenMemHandle(h, self._rt.cudaIpcMemLazyEnablePeerAccess)
        if err != self._rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"ipc heap: cudaIpcOpenMemHandle {err}")
        self._opened.append(int(ptr))
        return int(ptr)


class PeerComm:
    """One rank's view of the symmetric heap: named buffers, peer pointer arrays, flags."""

    def __init__(self, tp: int, rank: int, device, provider="symmetric_memory", group=None, scatter: bool = False,
                 nvls: bool = False):
        if not 1 <= tp <= 8:
            raise ValueError(f"peer boundaries support 1 <= tp <= 8, got {tp}")
        self.tp, self.rank = tp, rank
        self.dev = torch.device(device)
        self.provider = provider
        self.group = group
        # scatter=False (default): the GEMM stores locally and the boundary kernel pulls every rank's
        # bf16 partial (incoming link direction) while pushing a / dP (outgoing) — both NVLink
        # directions busy at once. scatter=True: the producing GEMM reduce-adds its output into the
        # owning ranks' fp32 buffers tile by tile (btp_gemm_scatter: GEMM + reduce-scatter in one
        # kernel, the transfer overlapped with the MMA) — but fp32 (sm_100a has no bf16 tensor
        # reduce) doubles the reduce-scatter bytes and both halves then use the outgoing direction,
        # so it only wins when the GEMM is long against the transfer.
        self.scatter = scatter
        if nvls and scatter:
            raise ValueError("nvls and scatter are alternative boundary forms")
        if provider == "local_multicast" and tp != 1:
            raise ValueError("the local multicast heap has one member: tp must be 1")
        self.nvls = nvls or provider == "local_multicast"
        self.mc_base = 0
        self.heap = None
        self._hptrs: dict[str, list[int]] = {}
        self._bufs: dict[str, torch.Tensor] = {}
        self._ptrs: dict[str, torch.Tensor] = {}
        self.epoch = torch.zeros(N_SLOTS, dtype=torch.int32, device=self.dev)

    # ------------------------------------------------------------------ heap
    def setup(self, specs) -> None:
        """specs: ordered [(name, shape, dtype)], identical on every rank. Allocates the heap,
        exchanges bases, zeroes the flags, and synchronises the ranks once."""
        layout, off = [], N_SLOTS * self.tp * 4
        off = -(-off // _ALIGN) * _ALIGN
        for name, shape, dtype in specs:
            n = 1
            for s in shape:
                n *= int(s)
            nbytes = n * torch.empty((), dtype=dtype).element_size()
            layout.append((name, tuple(shape), dtype, off, nbytes))
            off = -(-(off + nbytes) // _ALIGN) * _ALIGN
        total = off
        if isinstance(self.provider, VirtualPeers):
            self.heap = torch.empty(total, dtype=torch.uint8, device=self.dev)
            self.heap.zero_()  # flags, and the reduce-add targets of the scatter GEMMs
            torch.cuda.synchronize(self.dev)
            bases = self.provider.exchange(self.rank, self.heap.data_ptr())
        elif self.provider == "symmetric_memory":
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            self.heap = symm_mem.empty(total, dtype=torch.uint8, device=self.dev)
            self.heap.zero_()  # flags, and the reduce-add targets of the scatter GEMMs
            torch.cuda.synchronize(self.dev)
            group = self.group if self.group is not None else dist.group.WORLD
            hdl = symm_mem.rendezvous(self.heap, group)
            bases = [int(p) for p in hdl.buffer_ptrs]
            if self.nvls:
                self.mc_base = int(hdl.multicast_ptr)
                if not self.mc_base:
                    raise RuntimeError("symmetric memory returned no multicast address (NVLS unavailable)")
            self._symm = hdl
            dist.barrier(group=group)  # every rank's flags are zero before anyone signals
        elif self.provider == "cuda_ipc":
            import torch.distributed as dist

            self._ipc = IpcHeap(total, self.dev)
            self.heap = self._ipc.tensor
            self.heap.zero_()
            torch.cuda.synchronize(self.dev)
            group = self.group if self.group is not None else dist.group.WORLD
            handles = [None] * self.tp
            dist.all_gather_object(handles, self._ipc.handle(), group=group)
            bases = [self._ipc.ptr if j == self.rank else self._ipc.open(handles[j]) for j in range(self.tp)]
            dist.barrier(group=group)  # every rank's flags are zero before anyone signals
        elif self.provider == "local_multicast":
            self._mc_heap = LocalMulticastHeap(total, self.dev)
            self.heap = self._mc_heap.tensor
            self.heap.zero_()
            torch.cuda.synchronize(self.dev)
            bases, self.mc_base = [self.heap.data_ptr()], self._mc_heap.mc_ptr
        else:
            raise ValueError(f"unknown peer provider {self.provider!r}")
        if len(bases) != self.tp:
            raise RuntimeError(f"peer heap rendezvous returned {len(bases)} bases for tp={self.tp}")
        self.bases = bases
        self._flags_ptrs = torch.tensor(bases, dtype=torch.int64, device=self.dev)
        self._offsets = {}
        for name, shape, dtype, o, nbytes in layout:
            self._offsets[name] = o
            self._bufs[name] = self.heap[o:o + nbytes].view(dtype).view(shape)
            self._hptrs[name] = [b + o for b in bases]
            self._ptrs[name] = torch.tensor(self._hptrs[name], dtype=torch.int64, device=self.dev)
        torch.cuda.synchronize(self.dev)

    def has(self, name: str) -> bool:
        return name in self._bufs

    def buf(self, name: str) -> torch.Tensor:
        return self._bufs[name]

    def ptrs(self, name: str):
        return ctypes.c_void_p(self._ptrs[name].data_ptr())

    def mc(self, name: str):
        """Multicast address of buffer `name` (nvls only)."""
        if not self.mc_base:
            raise RuntimeError("this peer heap has no multicast mapping")
        return ctypes.c_void_p(self.mc_base + self._offsets[name])

    def host_ptrs(self, name: str) -> list[int]:
        """Every rank's address of buffer `name`, rank order (host ints, for tensor maps)."""
        return self._hptrs[name]

    # ------------------------------------------------------------------ signals
    def signal(self, slot: int) -> None:
        _native.call("btp_peer_signal", ctypes.c_void_p(self._flags_ptrs.data_ptr()),
                     ctypes.c_void_p(self.epoch.data_ptr()), slot, self.rank, self.tp, _stream())

    def wait(self, slot: int) -> None:
        _native.call("btp_peer_wait", ctypes.c_void_p(self.heap.data_ptr()), ctypes.c_void_p(self.epoch.data_ptr()),
                     slot, self.tp, _stream())

    def exchange(self, slot: int = READY) -> None:
        """signal + wait: a device-side barrier across the ranks on the current stream."""
        self.signal(slot)
        self.wait(slot)


def boundary_fwd(pc: PeerComm, P_name, ss_name, T, W, r, variant, d, eps, z_own, s_own, a_name) -> None:
    if pc.nvls:
        _native.call("btp_peer_boundary_fwd_nvls", pc.mc(P_name), pc.mc(ss_name) if ss_name else None, pc.tp,
                     pc.rank, T, W, r, variant, d, ctypes.c_float(eps), ctypes.c_void_p(z_own.data_ptr()),
                     ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None, pc.mc(a_name), _stream())
        return
    _native.call("btp_peer_boundary_fwd", pc.ptrs(P_name), pc.ptrs(ss_name) if ss_name else None, pc.tp, pc.rank,
                 T, W, r, variant, d, ctypes.c_float(eps), ctypes.c_void_p(z_own.data_ptr()),
                 ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None, pc.ptrs(a_name), _stream())


def boundary_bwd(pc: PeerComm, da_name, T, W, r, variant, d, z_own, s_own, dP_name, dss_name) -> None:
    if pc.nvls:
        _native.call("btp_peer_boundary_bwd_nvls", pc.mc(da_name), pc.tp, pc.rank, T, W, r, variant, d,
                     ctypes.c_void_p(z_own.data_ptr()),
                     ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None, pc.mc(dP_name),
                     pc.mc(dss_name) if dss_name else None, _stream())
        return
    _native.call("btp_peer_boundary_bwd", pc.ptrs(da_name), pc.tp, pc.rank, T, W, r, variant, d,
                 ctypes.c_void_p(z_own.data_ptr()), ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None,
                 pc.ptrs(dP_name), pc.ptrs(dss_name) if dss_name else None, _stream())


def boundary_fwd_local(pc: PeerComm, R_name, ss_name, T, W, r, variant, d, eps, z_own, s_own, a_name) -> None:
    _native.call("btp_peer_boundary_fwd_local", ctypes.c_void_p(pc.buf(R_name).data_ptr()),
                 pc.ptrs(ss_name) if ss_name else None, pc.tp, pc.rank, T, W, r, variant, d, ctypes.c_float(eps),
                 ctypes.c_void_p(z_own.data_ptr()), ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None,
                 pc.ptrs(a_name), _stream())


def boundary_bwd_local(pc: PeerComm, R_name, T, W, r, variant, d, z_own, s_own, dP_name, dss_name) -> None:
    _native.call("btp_peer_boundary_bwd_local", ctypes.c_void_p(pc.buf(R_name).data_ptr()), pc.tp, pc.rank, T, W, r,
                 variant, d, ctypes.c_void_p(z_own.data_ptr()),
                 ctypes.c_void_p(s_own.data_ptr()) if s_own is not None else None, pc.ptrs(dP_name),
                 pc.ptrs(dss_name) if dss_name else None, _stream())
