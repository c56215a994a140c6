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

__device__ __forceinline__ float silu_acc(float x) { return x * sigmoidf_safe(x); }

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

// Forward boundary: one warp per owned row; lane work units = 8 "u" + 8 "v" columns (cola) or 8
// columns (svd) of one projection.
// kLocal: the partials were already reduce-added into this rank's owned rows R_own [rows_own, W]
// by the other ranks' scatter GEMMs (btp_gemm_scatter): read them locally (and re-zero them for the
// next use) instead of pulling every rank's P.
__device__ __forceinline__ void own_sum8(float* R_own, long long off, float (&acc)[8]) {
  float4* p = reinterpret_cast<float4*>(R_own + off);
  const float4 a = __ldcv(p), b = __ldcv(p + 1);
  acc[0] = a.x; acc[1] = a.y; acc[2] = a.z; acc[3] = a.w; acc[4] = b.x; acc[5] = b.y; acc[6] = b.z; acc[7] = b.w;
  p[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  p[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

template <bool kLocal>
__global__ void __launch_bounds__(256) peer_boundary_fwd_kernel(
    const bf16* const* __restrict__ P_peers, float* __restrict__ R_own, const float* const* __restrict__ ss_peers,
    int tp, int row0, int rows_own, int W, int r, int variant, float inv_d, float eps, bf16* __restrict__ z_own,
    float* __restrict__ s_own, bf16* const* __restrict__ a_peers) {
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < rows_own; i += gridDim.x * warps) {
    const long long row = row0 + i;
    float s = 1.0f;
    if (ss_peers != nullptr) {
      float ss = 0.f;
      for (int j = 0; j < tp; ++j) ss += __ldcv(ss_peers[j] + row);
      s = sqrtf(ss * inv_d + eps);
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
        if constexpr (kLocal) {
          own_sum8(R_own, (long long)i * W + cu, zu);
          own_sum8(R_own, (long long)i * W + cv, zv);
        } else {
          pull_sum8(P_peers, tp, row * W + cu, zu);
          pull_sum8(P_peers, tp, row * W + cv, zv);
        }
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
          au[e] = silu_acc(zu[e]) * zv[e];
          av[e] = silu_acc(zv[e]) * zu[e];
        }
        const uint4 pu = pack8(au), pv = pack8(av);
        for (int j = 0; j < tp; ++j) {
          *reinterpret_cast<uint4*>(a_peers[j] + row * W + cu) = pu;
          *reinterpret_cast<uint4*>(a_peers[j] + row * W + cv) = pv;
        }
      } else {
        const int c = p * r + g * 8;
        float z[8];
        if constexpr (kLocal) own_sum8(R_own, (long long)i * W + c, z);
        else pull_sum8(P_peers, tp, row * W + c, z);
#pragma unroll
        for (int e = 0; e < 8; ++e) z[e] *= inv;
        const uint4 wz = pack8(z);
        *reinterpret_cast<uint4*>(z_own + (long long)i * W + c) = wz;
        for (int j = 0; j < tp; ++j) *reinterpret_cast<uint4*>(a_peers[j] + row * W + c) = wz;
      }
    }
  }
  __threadfence_system();  // pushes visible system-wide before the "done" signal
}

template <bool kLocal>
__global__ void __launch_bounds__(256) peer_boundary_bwd_kernel(
    const bf16* const* __restrict__ da_peers, float* __restrict__ R_own, int tp, int row0, int rows_own, int W, int r,
    int variant, float inv_d,
    const bf16* __restrict__ z_own, const float* __restrict__ s_own, bf16* const* __restrict__ dP_peers,
    float* const* __restrict__ dss_peers) {
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
        if constexpr (kLocal) {
          own_sum8(R_own, (long long)i * W + cu, du_);
          own_sum8(R_own, (long long)i * W + cv, dv_);
        } else {
          pull_sum8(da_peers, tp, row * W + cu, du_);
          pull_sum8(da_peers, tp, row * W + cv, dv_);
        }
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
        const uint4 pu = pack8(gu), pv = pack8(gv);
        for (int j = 0; j < tp; ++j) {
          *reinterpret_cast<uint4*>(dP_peers[j] + row * W + cu) = pu;
          *reinterpret_cast<uint4*>(dP_peers[j] + row * W + cv) = pv;
        }
      } else {
        const int c = p * r + g * 8;
        float dd[8], zz[8];
        if constexpr (kLocal) own_sum8(R_own, (long long)i * W + c, dd);
        else pull_sum8(da_peers, tp, row * W + c, dd);
        unpack8(*reinterpret_cast<const uint4*>(z_own + (long long)i * W + c), zz);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dot = fmaf(dd[e], zz[e], dot);
          dd[e] *= inv;
        }
        const uint4 pd = pack8(dd);
        for (int j = 0; j < tp; ++j) *reinterpret_cast<uint4*>(dP_peers[j] + row * W + c) = pd;
      }
    }
    dot = warp_sum32(dot);
    if (lane == 0 && dss_peers != nullptr && s_own != nullptr) {
      const float v = -dot * inv * inv * 0.5f * inv_d;
      for (int j = 0; j < tp; ++j) dss_peers[j][row] = v;
    }
  }
  __threadfence_system();
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
  if (R_own != nullptr)
    peer_boundary_fwd_kernel<true><<<rows_grid(rows_own), 256, 0, st>>>(
        nullptr, static_cast<float*>(R_own), ss_peers, tp, rank * rows_own, rows_own, W, r, variant, 1.0f / (float)d,
        eps, static_cast<bf16*>(z_own), s_own, reinterpret_cast<bf16* const*>(a_peers));
  else
    peer_boundary_fwd_kernel<false><<<rows_grid(rows_own), 256, 0, st>>>(
        reinterpret_cast<const bf16* const*>(P_peers), nullptr, ss_peers, tp, rank * rows_own, rows_own, W, r, variant,
        1.0f / (float)d, eps, static_cast<bf16*>(z_own), s_own, reinterpret_cast<bf16* const*>(a_peers));
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int peer_boundary_bwd(const void* const* da_peers, int tp, int rank, int T, int W, int r, int variant, int d,
                      const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                      cudaStream_t st, void* R_own) {
  if (int rc = check_geometry(tp, rank, T, W, r, variant)) return rc;
  if (d <= 0 || !z_own || !dP_peers || (!da_peers && !R_own) || !a16p(z_own)) return BTP_ERR_DIM;
  const int rows_own = T / tp;
  if (R_own != nullptr)
    peer_boundary_bwd_kernel<true><<<rows_grid(rows_own), 256, 0, st>>>(
        nullptr, static_cast<float*>(R_own), tp, rank * rows_own, rows_own, W, r, variant, 1.0f / (float)d,
        static_cast<const bf16*>(z_own), s_own, reinterpret_cast<bf16* const*>(dP_peers), dss_peers);
  else
    peer_boundary_bwd_kernel<false><<<rows_grid(rows_own), 256, 0, st>>>(
        reinterpret_cast<const bf16* const*>(da_peers), nullptr, tp, rank * rows_own, rows_own, W, r, variant,
        1.0f / (float)d, static_cast<const bf16*>(z_own), s_own, reinterpret_cast<bf16* const*>(dP_peers), dss_peers);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

}  // namespace btp
