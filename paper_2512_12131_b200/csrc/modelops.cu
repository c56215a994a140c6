// Model-boundary kernels around the stack of BTP blocks: the d-sharded
// token embedding that feeds the first block's row-split down-projection, and the fused
// softmax cross-entropy (loss + logits gradient) of the replicated LM head.
//
// All HBM-bound: 128-bit accesses of 8 elements, fp32 math. The embedding backward
// accumulates rows of the table gradient with fp32 atomics (repeated token ids collide; the
// summation order across them is not fixed). The cross-entropy reduction is per row, one block
// per row, with fixed-order warp/block reductions (deterministic).
#include <cuda_runtime.h>

#include "btp_internal.h"
#include "ptx.cuh"

namespace btp {

using bf16 = __nv_bfloat16;

namespace {

template <typename T>
struct Acc8;

template <>
struct Acc8<bf16> {
  __device__ static __forceinline__ void ld(const bf16* p, float (&f)[8]) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    f[0] = bf16_lo(w.x); f[1] = bf16_hi(w.x); f[2] = bf16_lo(w.y); f[3] = bf16_hi(w.y);
    f[4] = bf16_lo(w.z); f[5] = bf16_hi(w.z); f[6] = bf16_lo(w.w); f[7] = bf16_hi(w.w);
  }
  __device__ static __forceinline__ void st(bf16* p, const float (&f)[8]) {
    *reinterpret_cast<uint4*>(p) =
        make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
  }
};

template <>
struct Acc8<float> {
  __device__ static __forceinline__ void ld(const float* p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
  __device__ static __forceinline__ void st(float* p, const float (&f)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
  }
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_add(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace

// out[t, :] = table[ids[t], col0 : col0 + width]   (this rank's d-shard of the embedding)
template <typename T>
__global__ void __launch_bounds__(256) embedding_fwd_kernel(const int* __restrict__ ids, const T* __restrict__ table,
                                                            long long ldt, int vocab, int col0, T* __restrict__ out,
                                                            long long ldo, int rows, int width, int* __restrict__ bad) {
  const int per_row = width >> 3;
  const long long total = (long long)rows * per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i / per_row);
    const int c = (int)(i - (long long)t * per_row) * 8;
    const int id = __ldg(ids + t);
    float f[8];
    if (id < 0 || id >= vocab) {  // out-of-range id: zero row + flag (reported by the launcher's caller)
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = 0.f;
      if (bad) *bad = 1;
    } else {
      Acc8<T>::ld(table + (long long)id * ldt + col0 + c, f);
    }
    Acc8<T>::st(out + (long long)t * ldo + c, f);
  }
}

// dtable[ids[t], c] += dx[t, c]   (fp32 gradient of this rank's shard, zero-initialised)
template <typename T>
__global__ void __launch_bounds__(256) embedding_bwd_kernel(const int* __restrict__ ids, const T* __restrict__ dx,
                                                            long long lddx, int vocab, float* __restrict__ dtable,
                                                            long long ldg, int rows, int width) {
  const int per_row = width >> 3;
  const long long total = (long long)rows * per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i / per_row);
    const int c = (int)(i - (long long)t * per_row) * 8;
    const int id = __ldg(ids + t);
    if (id < 0 || id >= vocab) continue;
    float f[8];
    Acc8<T>::ld(dx + (long long)t * lddx + c, f);
    float* g = dtable + (long long)id * ldg + c;
#pragma unroll
    for (int j = 0; j < 8; ++j) atomicAdd(g + j, f[j]);
  }
}

// One block per row of logits [rows, V]:
//   m = max_j l_j ; lse = m + log(sum_j exp(l_j - m)) ; loss[t] = lse - l[target]
//   dlogits[t, j] = scale * (exp(l_j - lse) - [j == target])      (dlogits may alias logits)
// Rows whose target is < 0 (ignore index) get loss 0 and a zero gradient.
template <typename T>
__global__ void __launch_bounds__(512) cross_entropy_kernel(const T* logits, long long ldl,
                                                            const int* __restrict__ targets, int vocab,
                                                            float* __restrict__ loss_rows, T* dlogits, long long ldd,
                                                            float scale) {
  __shared__ float red_m[16], red_s[16];
  const int t = blockIdx.x;
  const T* row = logits + (long long)t * ldl;
  const int nch = vocab >> 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // pass 1: per-thread online (max, sum of exp)
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    float f[8];
    Acc8<T>::ld(row + c * 8, f);
    float cm = f[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) cm = fmaxf(cm, f[j]);
    const float nm = fmaxf(m, cm);
    float acc = s * __expf(m - nm);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __expf(f[j] - nm);
    m = nm;
    s = acc;
  }
  // combine (max, sum) across the block in a fixed order
  float wm = warp_max(m);
  s = (m == -INFINITY) ? 0.f : s * __expf(m - wm);
  s = warp_add(s);
  if (lane == 0) {
    red_m[warp] = wm;
    red_s[warp] = s;
  }
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < nwarps; ++w) M = fmaxf(M, red_m[w]);
  float S = 0.f;
  for (int w = 0; w < nwarps; ++w) S += (red_m[w] == -INFINITY) ? 0.f : red_s[w] * __expf(red_m[w] - M);
  const float lse = M + __logf(S);
  const int tgt = targets[t];
  if (threadIdx.x == 0) {
    float lt = 0.f;
    if (tgt >= 0 && tgt < vocab) {
      float f[8];
      Acc8<T>::ld(row + (tgt & ~7), f);
      lt = f[tgt & 7];
    }
    loss_rows[t] = (tgt >= 0 && tgt < vocab) ? (lse - lt) : 0.f;
  }
  if (dlogits == nullptr) return;
  __syncthreads();  // the target logit is read before an aliasing gradient overwrites it
  T* drow = dlogits + (long long)t * ldd;
  const bool live = tgt >= 0 && tgt < vocab;
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    float f[8];
    Acc8<T>::ld(row + c * 8, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p = live ? __expf(f[j] - lse) : 0.f;
      f[j] = scale * (p - ((live && c * 8 + j == tgt) ? 1.f : 0.f));
    }
    Acc8<T>::st(drow + c * 8, f);
  }
}

static inline bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static inline int grid_cap(long long items) {
  const long long want = (items + 255) / 256;
  const long long cap = (long long)num_sms_cached() * 16;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int embedding_fwd(const int* ids, const void* table, long long ldt, int vocab, int col0, void* out, long long ldo,
                  int rows, int width, int* bad, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0 || vocab <= 0 || col0 < 0) return BTP_ERR_DIM;
  if (width % 8 || ldt % 8 || ldo % 8 || col0 % 8 || !a16(table) || !a16(out)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_cap((long long)rows * width / 8);
  if (f32)
    embedding_fwd_kernel<float><<<grid, 256, 0, st>>>(ids, static_cast<const float*>(table), ldt, vocab, col0,
                                                      static_cast<float*>(out), ldo, rows, width, bad);
  else
    embedding_fwd_kernel<bf16><<<grid, 256, 0, st>>>(ids, static_cast<const bf16*>(table), ldt, vocab, col0,
                                                     static_cast<bf16*>(out), ldo, rows, width, bad);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int embedding_bwd(const int* ids, const void* dx, long long lddx, int vocab, float* dtable, long long ldg, int rows,
                  int width, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0 || vocab <= 0) return BTP_ERR_DIM;
  if (width % 8 || lddx % 8 || !a16(dx)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_cap((long long)rows * width / 8);
  if (f32)
    embedding_bwd_kernel<float><<<grid, 256, 0, st>>>(ids, static_cast<const float*>(dx), lddx, vocab, dtable, ldg,
                                                      rows, width);
  else
    embedding_bwd_kernel<bf16><<<grid, 256, 0, st>>>(ids, static_cast<const bf16*>(dx), lddx, vocab, dtable, ldg, rows,
                                                     width);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int cross_entropy(const void* logits, long long ldl, const int* targets, int vocab, float* loss_rows, void* dlogits,
                  long long ldd, int rows, float scale, cudaStream_t st, bool f32) {
  if (rows <= 0 || vocab <= 0) return BTP_ERR_DIM;
  if (vocab % 8 || ldl % 8 || (dlogits && ldd % 8) || !a16(logits) || (dlogits && !a16(dlogits)))
    return BTP_ERR_ALIGNMENT;
  const int threads = vocab >= 4096 ? 512 : 128;
  if (f32)
    cross_entropy_kernel<float><<<rows, threads, 0, st>>>(static_cast<const float*>(logits), ldl, targets, vocab,
                                                          loss_rows, static_cast<float*>(dlogits), ldd, scale);
  else
    cross_entropy_kernel<bf16><<<rows, threads, 0, st>>>(static_cast<const bf16*>(logits), ldl, targets, vocab,
                                                         loss_rows, static_cast<bf16*>(dlogits), ldd, scale);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

}  // namespace btp
