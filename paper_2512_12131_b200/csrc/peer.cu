// BTP chunk boundaries over NVLink/NVSwitch peer memory: the all-reduce that
// follows every row-parallel down-projection is restated as
//
//     reduce-scatter (pull) -> fix-up + sigma on the rows this rank owns -> all-gather (push)
//
// in ONE kernel per chunk, so the normalisation fix-up and the crossgate activation ride the
// collective instead of costing their own HBM pass, and no NCCL kernel competes for SMs.
//
// Every rank owns T/tp consecutive rows. Forward (btp_peer_boundary_fwd), per owned row t:
//     P  = sum_j P_j[t, :]                       (bf16 partials of all ranks, fp32 sum, rank order 0..tp-1:
//                                                  every rank computes bit-identical values)
//     s  = sqrt(sum_j ss_j[t] / d + eps)          (online-norm rider; absent on o / down chunks: s = 1)
//     z  = bf16(P / s) -> z_own (kept for backward, owned rows only)
//     a  = sigma(z)    -> pushed into a_j[t, :] of EVERY rank j (the up-projection's replicated input)
// Backward (btp_peer_boundary_bwd), per owned row t:
//     da = sum_j da_j[t, :]                       (the up-projection dgrad partials)
//     dz = sigma'(z) da ; dP = dz / s -> pushed to every rank ; dss = -<dz, z>/(2 s^2 d) -> pushed
// Bytes crossing NVLink per rank and direction: (tp-1)/tp * T * W * 2 pulled + the same pushed,
// i.e. a ring all-reduce's 2(tp-1)/tp * T * W * 2 — with the fix-up fused in.
//
// Ordering: a rank signals "ready" after producing its partial (btp_peer_signal, release at system
// scope), and waits (btp_peer_wait, acquire) for every rank's "ready" before pulling; after pushing
// it signals "done" and waits for every rank's "done" before the consumer reads what was pushed.
// Flags are monotone per-slot epochs kept in device memory (graph-replay safe): rank r's k-th
// signal on slot s stores k into flags_j[s * tp + r] of every rank j.
//
// The peer pointer arrays are device arrays of tp pointers (rank order) into each rank's symmetric
// buffer: torch symmetric-memory (cuMem IPC over NVLink) across processes on the box, or tp
// buffers of one device in the single-GPU multi-rank test.
#include <type_traits>
#include <cuda_runtime.h>

#include <cstdio>

#include "btp_internal.h"
#include "ptx.cuh"

namespace btp {

using bf16 = __nv_bfloat16;

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void unpack8(const uint4& w, float (&f)[8]) {
  f[0] = bf16_lo(w.x); f[1] = bf16_hi(w.x); f[2] = bf16_lo(w.y); f[3] = bf16_hi(w.y);
  f[4] = bf16_lo(w.z); f[5] = bf16_hi(w.z); f[6] = bf16_lo(w.w); f[7] = bf16_hi(w.w);
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}


__device__ __forceinline__ float warp_sum32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kMaxTP = 8;

// sum over ranks (fixed order) of the 8-element chunk at element offset `off` of every peer's row
__device__ __forceinline__ void pull_sum8(const bf16* const* peers, int tp, long long off, float (&acc)[8]) {
  uint4 w[kMaxTP];
#pragma unroll
  for (int j = 0; j < kMaxTP; ++j)
    if (j < tp) w[j] = __ldcv(reinterpret_cast<const uint4*>(peers[j] + off));  // all loads in flight first
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxTP; ++j) {
    if (j < tp) {
      float f[8];
      unpack8(w[j], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += f[e];
    }
  }
}

}  // namespace

__global__ void peer_signal_kernel(uint32_t* const* __restrict__ peer_flags, uint32_t* __restrict__ epoch, int slot,
                                   int rank, int tp) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  const uint32_t e = epoch[slot] + 1u;
  epoch[slot] = e;
  for (int j = 0; j < tp; ++j) st_release_sys(peer_flags[j] + slot * tp + rank, e);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A peer that never arrives (a crashed rank) must not hang the GPU: after kPeerTimeoutNs the wait
// traps, which fails the stream with a launch error the host sees.
constexpr uint64_t kPeerTimeoutNs = 120ull * 1000000000ull;

__global__ void peer_wait_kernel(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ epoch, int slot,
                                 int tp) {
  const int j = threadIdx.x;
  if (j < tp) {
    const uint32_t e = epoch[slot];
    const uint64_t t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(flags + slot * tp + j) - e) < 0) {
      __nanosleep(100);
      if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
        printf("btp_peer_wait: rank %d never reached epoch %u on slot %d\n", j, e, slot);
        __trap();
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

// The boundary kernels are written once over "where the partials come from" and "where the
// results go" (the policies below); one warp per owned row, lane work units = 8 "u" + 8 "v"
// columns (cola) or 8 columns (svd) of one projection. Sources of the reduced row:
//   PullRows   — sum every rank's bf16 partial over NVLink (fp32 accumulation)
//   LocalRows  — the partials were already reduce-added into this rank's owned rows R_own
//                [rows_own, W] by the other ranks' scatter GEMMs (btp_gemm_scatter): read them
//                locally and re-zero them for the next use
//   McRows     — NVLS: multimem.ld_reduce on the multicast address, the switch sums (acc::f32)
// Destinations of a / dP / dss: PushRows (a store into every rank's copy) or McRows (one
// multimem.st, replicated by the switch). Only these primitives differ between the forms, so the
// NVLS kernels share every line of fix-up / sigma math with the pull kernels the tests pin.
namespace {

struct PullRows {
  const bf16* const* src;
  int tp;
  __device__ __forceinline__ void sum8(long long g, long long, float (&f)[8]) const { pull_sum8(src, tp, g, f); }
};

struct LocalRows {
  float* R_own;
  __device__ __forceinline__ void sum8(long long, long long l, float (&f)[8]) const {
    float4* q = reinterpret_cast<float4*>(R_own + l);
    const float4 a = __ldcv(q), b = __ldcv(q + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    q[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    q[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
};

struct PushRows {
  bf16* const* dst;
  int tp;
  __device__ __forceinline__ void store8(long long g, const uint4& w) const {
    for (int j = 0; j < tp; ++j) *reinterpret_cast<uint4*>(dst[j] + g) = w;
  }
};

struct McRows {  // NVLS multicast address of a bf16 [T, W] buffer
  bf16* mc;
  __device__ __forceinline__ void sum8(long long g, long long, float (&f)[8]) const {
    uint32_t a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(mc + g)
                 : "memory");
    unpack8(make_uint4(a, b, c, d), f);
  }
  __device__ __forceinline__ void store8(long long g, const uint4& w) const {
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc + g), "r"(w.x), "r"(w.y),
                 "r"(w.z), "r"(w.w)
                 : "memory");
  }
};

struct PullStat {  // per-row fp32 statistic, one copy per rank
  const float* const* src;
  int tp;
  __device__ __forceinline__ bool on() const { return src != nullptr; }
  __device__ __forceinline__ float sum(long long row) const {
    float v = 0.f;
    for (int j = 0; j < tp; ++j) v += __ldcv(src[j] + row);
    return v;
  }
};

struct PushStat {
  float* const* dst;
  int tp;
  __device__ __forceinline__ bool on() const { return dst != nullptr; }
  __device__ __forceinline__ void store(long long row, float v) const {
    for (int j = 0; j < tp; ++j) dst[j][row] = v;
  }
};

struct McStat {
  float* mc;
  __device__ __forceinline__ bool on() const { return mc != nullptr; }
  __device__ __forceinline__ float sum(long long row) const {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + row) : "memory");
    return v;
  }
  __device__ __forceinline__ void store(long long row, float v) const {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc + row), "f"(v) : "memory");
  }
};

// every store of this kernel (peer-mapped or multicast) visible system-wide before the "done" signal
template <class Dst>
__device__ __forceinline__ void release_pushes() {
  __threadfence_system();
  if constexpr (std::is_same_v<Dst, McRows>)
    asm volatile("fence.proxy.alias;" ::: "memory");  // multicast vs unicast aliases of the same pages
}

}  // namespace

template <class Src, class Stat, class Dst>
__global__ void __launch_bounds__(256) peer_boundary_fwd_kernel(Src P, Stat ss, int row0, int rows_own, int W, int r,
                                                                int variant, float inv_d, float eps,
                                                                bf16* __restrict__ z_own, float* __restrict__ s_own,
                                                                Dst A) {
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < rows_own; i += gridDim.x * warps) {
    const long long row = row0 + i;
    float s = 1.0f;
    if (ss.on()) {
      s = sqrtf(ss.sum(row) * inv_d + eps);
      if (lane == 0 && s_own != nullptr) s_own[i] = s;
    }
    const float inv = 1.0f / s;
    const int per_proj = variant == 1 ? (r >> 4) : (r >> 3);
    const int units = per_proj * (W / r);
    for (int u = lane; u < units; u += 32) {
      const int p = u / per_proj, g = u - p * per_proj;
      if (variant == 1) {
        const int cu = p * r + g * 8, cv = cu + (r >> 1);
        float zu[8], zv[8];
        P.sum8(row * W + cu, (long long)i * W + cu, zu);
        P.sum8(row * W + cv, (long long)i * W + cv, zv);
#pragma unroll
        for (int e = 0; e < 8; ++e) { zu[e] *= inv; zv[e] *= inv; }
        const uint4 wu = pack8(zu), wv = pack8(zv);
        *reinterpret_cast<uint4*>(z_own + (long long)i * W + cu) = wu;
        *reinterpret_cast<uint4*>(z_own + (long long)i * W + cv) = wv;
        unpack8(wu, zu);  // sigma acts on the stored (rounded) z, like btp_fixup_sigma
        unpack8(wv, zv);
        float au[8], av[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          au[e] = silu_crossgate<__nv_bfloat16>(zu[e]) * zv[e];
          av[e] = silu_crossgate<__nv_bfloat16>(zv[e]) * zu[e];
        }
        A.store8(row * W + cu, pack8(au));
        A.store8(row * W + cv, pack8(av));
      } else {
        const int c = p * r + g * 8;
        float z[8];
        P.sum8(row * W + c, (long long)i * W + c, z);
#pragma unroll
        for (int e = 0; e < 8; ++e) z[e] *= inv;
        const uint4 wz = pack8(z);
        *reinterpret_cast<uint4*>(z_own + (long long)i * W + c) = wz;
        A.store8(row * W + c, wz);
      }
    }
  }
  release_pushes<Dst>();
}

template <class Src, class Dst, class DssDst>
__global__ void __launch_bounds__(256) peer_boundary_bwd_kernel(Src dA, int row0, int rows_own, int W, int r,
                                                                int variant, float inv_d,
                                                                const bf16* __restrict__ z_own,
                                                                const float* __restrict__ s_own, Dst dP, DssDst dss) {
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < rows_own; i += gridDim.x * warps) {
    const long long row = row0 + i;
    const float s = s_own != nullptr ? s_own[i] : 1.0f;
    const float inv = 1.0f / s;
    const int per_proj = variant == 1 ? (r >> 4) : (r >> 3);
    const int units = per_proj * (W / r);
    float dot = 0.f;
    for (int u = lane; u < units; u += 32) {
      const int p = u / per_proj, g = u - p * per_proj;
      if (variant == 1) {
        const int cu = p * r + g * 8, cv = cu + (r >> 1);
        float du_[8], dv_[8], zu[8], zv[8];
        dA.sum8(row * W + cu, (long long)i * W + cu, du_);
        dA.sum8(row * W + cv, (long long)i * W + cv, dv_);
        unpack8(*reinterpret_cast<const uint4*>(z_own + (long long)i * W + cu), zu);
        unpack8(*reinterpret_cast<const uint4*>(z_own + (long long)i * W + cv), zv);
        float gu[8], gv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float su = sigmoidf_safe(zu[e]), sv = sigmoidf_safe(zv[e]);
          const float dsu = su * (1.0f + zu[e] * (1.0f - su)), dsv = sv * (1.0f + zv[e] * (1.0f - sv));
          gu[e] = du_[e] * dsu * zv[e] + dv_[e] * zv[e] * sv;
          gv[e] = du_[e] * zu[e] * su + dv_[e] * dsv * zu[e];
          dot = fmaf(gu[e], zu[e], dot);
          dot = fmaf(gv[e], zv[e], dot);
          gu[e] *= inv;
          gv[e] *= inv;
        }
        dP.store8(row * W + cu, pack8(gu));
        dP.store8(row * W + cv, pack8(gv));
      } else {
        const int c = p * r + g * 8;
        float dd[8], zz[8];
        dA.sum8(row * W + c, (long long)i * W + c, dd);
        unpack8(*reinterpret_cast<const uint4*>(z_own + (long long)i * W + c), zz);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dot = fmaf(dd[e], zz[e], dot);
          dd[e] *= inv;
        }
        dP.store8(row * W + c, pack8(dd));
      }
    }
    dot = warp_sum32(dot);
    if (lane == 0 && dss.on() && s_own != nullptr) dss.store(row, -dot * inv * inv * 0.5f * inv_d);
  }
  release_pushes<Dst>();
}

static inline bool a16p(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static inline int rows_grid(int rows) {
  const int want = (rows + 7) / 8;
  const int cap = num_sms_cached() * 8;
  return want < cap ? (want > 0 ? want : 1) : cap;
}

int peer_signal(uint32_t* const* peer_flags, uint32_t* epoch, int slot, int rank, int tp, cudaStream_t st) {
  if (tp < 1 || tp > kMaxTP || rank < 0 || rank >= tp || slot < 0) return BTP_ERR_DIM;
  peer_signal_kernel<<<1, 32, 0, st>>>(peer_flags, epoch, slot, rank, tp);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int peer_wait(const uint32_t* flags, const uint32_t* epoch, int slot, int tp, cudaStream_t st) {
  if (tp < 1 || tp > kMaxTP || slot < 0) return BTP_ERR_DIM;
  peer_wait_kernel<<<1, 32, 0, st>>>(flags, epoch, slot, tp);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

static int check_geometry(int tp, int rank, int T, int W, int r, int variant) {
  if (tp < 1 || tp > kMaxTP || rank < 0 || rank >= tp || T <= 0 || W <= 0 || r <= 0) return BTP_ERR_DIM;
  if (T % tp) return BTP_ERR_DIVISIBILITY;
  if (variant != 0 && variant != 1) return BTP_ERR_DIM;
  if (W % r || r % (variant == 1 ? 16 : 8)) return BTP_ERR_DIVISIBILITY;
  return BTP_OK;
}

int peer_boundary_fwd(const void* const* P_peers, const float* const* ss_peers, int tp, int rank, int T, int W, int r,
                      int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                      cudaStream_t st, void* R_own) {
  if (int rc = check_geometry(tp, rank, T, W, r, variant)) return rc;
  if (d <= 0 || !z_own || !a_peers || (!P_peers && !R_own) || !a16p(z_own)) return BTP_ERR_DIM;
  const int rows_own = T / tp;
  const PullStat ss{ss_peers, tp};
  const PushRows A{reinterpret_cast<bf16* const*>(a_peers), tp};
  if (R_own != nullptr)
    peer_boundary_fwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
        LocalRows{static_cast<float*>(R_own)}, ss, rank * rows_own, rows_own, W, r, variant, 1.0f / (float)d, eps,
        static_cast<bf16*>(z_own), s_own, A);
  else
    peer_boundary_fwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
        PullRows{reinterpret_cast<const bf16* const*>(P_peers), tp}, ss, rank * rows_own, rows_own, W, r, variant,
        1.0f / (float)d, eps, static_cast<bf16*>(z_own), s_own, A);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int peer_boundary_bwd(const void* const* da_peers, int tp, int rank, int T, int W, int r, int variant, int d,
                      const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                      cudaStream_t st, void* R_own) {
  if (int rc = check_geometry(tp, rank, T, W, r, variant)) return rc;
  if (d <= 0 || !z_own || !dP_peers || (!da_peers && !R_own) || !a16p(z_own)) return BTP_ERR_DIM;
  const int rows_own = T / tp;
  const PushRows dP{reinterpret_cast<bf16* const*>(dP_peers), tp};
  const PushStat dss{dss_peers, tp};
  if (R_own != nullptr)
    peer_boundary_bwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
        LocalRows{static_cast<float*>(R_own)}, rank * rows_own, rows_own, W, r, variant, 1.0f / (float)d,
        static_cast<const bf16*>(z_own), s_own, dP, dss);
  else
    peer_boundary_bwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
        PullRows{reinterpret_cast<const bf16* const*>(da_peers), tp}, rank * rows_own, rows_own, W, r, variant,
        1.0f / (float)d, static_cast<const bf16*>(z_own), s_own, dP, dss);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}


// ---------------------------------------------------------------------------------------------
// NVLS (NVLink SHARP) form of the boundaries: every rank's symmetric buffers are also bound to one
// NVSwitch multicast object, and the kernels use its multicast address *_mc:
//   multimem.ld_reduce ... add.acc::f32  — the switch sums the tp ranks' partials (fp32 accumulate)
//                                           and returns the owned row once: (T/tp)·W·2 B in per rank
//   multimem.st                          — one store of a / dP is replicated to every rank by the
//                                           switch: (T/tp)·W·2 B out per rank
// i.e. 2/tp of T·W·2 B per rank over NVLink instead of a ring's 2(tp-1)/tp. Same contract, flags
// and fix-up math as btp_peer_boundary_fwd / _bwd.
int peer_boundary_fwd_nvls(const void* P_mc, const float* ss_mc, int tp, int rank, int T, int W, int r, int variant,
                           int d, float eps, void* z_own, float* s_own, void* a_mc, cudaStream_t st) {
  if (int rc = check_geometry(tp, rank, T, W, r, variant)) return rc;
  if (d <= 0 || !z_own || !P_mc || !a_mc || !a16p(z_own) || !a16p(P_mc) || !a16p(a_mc)) return BTP_ERR_DIM;
  const int rows_own = T / tp;
  peer_boundary_fwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
      McRows{static_cast<bf16*>(const_cast<void*>(P_mc))}, McStat{const_cast<float*>(ss_mc)}, rank * rows_own,
      rows_own, W, r, variant, 1.0f / (float)d, eps, static_cast<bf16*>(z_own), s_own, McRows{static_cast<bf16*>(a_mc)});
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int peer_boundary_bwd_nvls(const void* dA_mc, int tp, int rank, int T, int W, int r, int variant, int d,
                           const void* z_own, const float* s_own, void* dP_mc, float* dss_mc, cudaStream_t st) {
  if (int rc = check_geometry(tp, rank, T, W, r, variant)) return rc;
  if (d <= 0 || !z_own || !dA_mc || !dP_mc || !a16p(z_own) || !a16p(dA_mc) || !a16p(dP_mc)) return BTP_ERR_DIM;
  const int rows_own = T / tp;
  peer_boundary_bwd_kernel<<<rows_grid(rows_own), 256, 0, st>>>(
      McRows{static_cast<bf16*>(const_cast<void*>(dA_mc))}, rank * rows_own, rows_own, W, r, variant, 1.0f / (float)d,
      static_cast<const bf16*>(z_own), s_own, McRows{static_cast<bf16*>(dP_mc)}, McStat{dss_mc});
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

}  // namespace btp
