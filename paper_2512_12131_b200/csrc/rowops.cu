// HBM-bound row/elementwise kernels of the BTP block: online RMSNorm + residual (K3),
// post-all-reduce fix-up + crossgate sigma (K4), SwiGLU (K5), and their backward passes.
//
// Every kernel is templated on the activation element type T: bf16 (the training path,
// 128-bit accesses of 8 elements) or fp32 (the parity mode, two 128-bit accesses per 8
// elements). Statistics and math are always fp32. Row reductions use one warp per row with
// shuffle reductions (no atomics), so every result is deterministic.
#include <cuda_runtime.h>

#include "btp_internal.h"
#include "ptx.cuh"

namespace btp {

using bf16 = __nv_bfloat16;

// ----------------------------------------------------------------------------- 8-wide access
template <typename T>
struct Vec8;

template <>
struct Vec8<bf16> {
  using Raw = uint4;
  __device__ static __forceinline__ Raw ld(const bf16* p) { return *reinterpret_cast<const uint4*>(p); }
  __device__ static __forceinline__ void st(bf16* p, const Raw& r) { *reinterpret_cast<uint4*>(p) = r; }
  __device__ static __forceinline__ void unpack(const Raw& w, float (&f)[8]) {
    f[0] = bf16_lo(w.x); f[1] = bf16_hi(w.x);
    f[2] = bf16_lo(w.y); f[3] = bf16_hi(w.y);
    f[4] = bf16_lo(w.z); f[5] = bf16_hi(w.z);
    f[6] = bf16_lo(w.w); f[7] = bf16_hi(w.w);
  }
  __device__ static __forceinline__ Raw pack(const float (&f)[8]) {
    return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
  }
};

template <>
struct Vec8<float> {
  struct Raw {
    float4 a, b;
  };
  __device__ static __forceinline__ Raw ld(const float* p) {
    return Raw{reinterpret_cast<const float4*>(p)[0], reinterpret_cast<const float4*>(p)[1]};
  }
  __device__ static __forceinline__ void st(float* p, const Raw& r) {
    reinterpret_cast<float4*>(p)[0] = r.a;
    reinterpret_cast<float4*>(p)[1] = r.b;
  }
  __device__ static __forceinline__ void unpack(const Raw& w, float (&f)[8]) {
    f[0] = w.a.x; f[1] = w.a.y; f[2] = w.a.z; f[3] = w.a.w;
    f[4] = w.b.x; f[5] = w.b.y; f[6] = w.b.z; f[7] = w.b.w;
  }
  __device__ static __forceinline__ Raw pack(const float (&f)[8]) {
    return Raw{make_float4(f[0], f[1], f[2], f[3]), make_float4(f[4], f[5], f[6], f[7])};
  }
};

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]) {
  Vec8<T>::unpack(Vec8<T>::ld(p), f);
}

template <typename T>
__device__ __forceinline__ void store8(T* p, const float (&f)[8]) {
  Vec8<T>::st(p, Vec8<T>::pack(f));
}

__device__ __forceinline__ void load_gamma8(const float* g, float (&f)[8]) {
  const float4 g0 = __ldg(reinterpret_cast<const float4*>(g));
  const float4 g1 = __ldg(reinterpret_cast<const float4*>(g + 4));
  f[0] = g0.x; f[1] = g0.y; f[2] = g0.z; f[3] = g0.w;
  f[4] = g1.x; f[5] = g1.y; f[6] = g1.z; f[7] = g1.w;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float silu_f(float x) { return x * sigmoidf_safe(x); }

// ----------------------------------------------------------------------------- K3 forward
// One warp per row; NCH = max 8-element chunks per lane held in registers.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) rmsnorm_residual_kernel(const T* __restrict__ x, long long ldx,
                                                               const T* __restrict__ branch, long long ldb,
                                                               T* __restrict__ x_out, long long ldo,
                                                               const float* __restrict__ gamma, T* __restrict__ n_out,
                                                               long long ldn, float* __restrict__ ss_out,
                                                               float* __restrict__ rl_out, int rows, int width,
                                                               float eps) {
  using V = Vec8<T>;
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nch = width >> 3;
  typename V::Raw keep[NCH];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = lane + 32 * i;
    if (c < nch) {
      typename V::Raw w = V::ld(x + (long long)row * ldx + c * 8);
      if (branch != nullptr) {
        float fx[8], fb[8];
        V::unpack(w, fx);
        load8(branch + (long long)row * ldb + c * 8, fb);
#pragma unroll
        for (int j = 0; j < 8; ++j) fx[j] += fb[j];
        w = V::pack(fx);
        if (x_out != nullptr) V::st(x_out + (long long)row * ldo + c * 8, w);
      }
      keep[i] = w;
      float f[8];
      V::unpack(w, f);  // statistics of the stored (rounded) value
#pragma unroll
      for (int j = 0; j < 8; ++j) ss = fmaf(f[j], f[j], ss);
    }
  }
  ss = warp_sum(ss);
  const float rl = sqrtf(ss / (float)width + eps);
  if (lane == 0) {
    if (ss_out) ss_out[row] = ss;
    if (rl_out) rl_out[row] = rl;
  }
  if (n_out == nullptr) return;
  const float inv = 1.0f / rl;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = lane + 32 * i;
    if (c < nch) {
      float f[8], g[8];
      V::unpack(keep[i], f);
      load_gamma8(gamma + c * 8, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = f[j] * g[j] * inv;
      store8(n_out + (long long)row * ldn + c * 8, f);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_apply_kernel(const T* __restrict__ x, long long ldx,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ ss_total, int d, float eps,
                                                            T* __restrict__ n_out, long long ldn,
                                                            float* __restrict__ rms_out, int rows, int width) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float s = sqrtf(ss_total[row] / (float)d + eps);
  if (lane == 0 && rms_out) rms_out[row] = s;
  const float inv = 1.0f / s;
  for (int c = lane; c < (width >> 3); c += 32) {
    float f[8], g[8];
    load8(x + (long long)row * ldx + c * 8, f);
    load_gamma8(gamma + c * 8, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * g[j] * inv;
    store8(n_out + (long long)row * ldn + c * 8, f);
  }
}

// ----------------------------------------------------------------------------- K4 forward
// Work item = (row, projection, group of 8 columns of the u half) for cola,
//             (row, projection, group of 8 columns) for svd.
// TIn: the reduced partial P's type — T, or fp32 when the boundary all-reduce ran in fp32 (one
// rounding of the cross-rank sum, here, instead of one per NCCL ring hop)
template <typename T, typename TIn = T>
__global__ void __launch_bounds__(256) fixup_sigma_kernel(const TIn* P, long long ldp, const float* __restrict__ ss_total,
                                                          int d, float eps, float* __restrict__ s_out, T* z_out,
                                                          long long ldz, T* __restrict__ a_out, long long lda,
                                                          int rows, int r, int nproj, int variant) {
  using V = Vec8<T>;
  const int per_proj = variant == 1 ? (r >> 4) : (r >> 3);
  const long long per_row = (long long)per_proj * nproj;
  const long long total = per_row * rows;
  const bool write_z = (z_out != nullptr) && (ss_total != nullptr || (const void*)z_out != (const void*)P);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / per_row);
    const int rem = (int)(idx - (long long)row * per_row);
    const int p = rem / per_proj;
    const int g = rem - p * per_proj;
    float inv = 1.0f;
    if (ss_total != nullptr) {
      const float s = sqrtf(ss_total[row] / (float)d + eps);
      inv = 1.0f / s;
      if (s_out != nullptr && p == 0 && g == 0) s_out[row] = s;
    }
    if (variant == 1) {
      const int cu = p * r + g * 8, cv = cu + (r >> 1);
      float u[8], v[8];
      load8(P + (long long)row * ldp + cu, u);
      load8(P + (long long)row * ldp + cv, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) { u[j] *= inv; v[j] *= inv; }
      const typename V::Raw zu = V::pack(u), zv = V::pack(v);
      if (write_z) {
        V::st(z_out + (long long)row * ldz + cu, zu);
        V::st(z_out + (long long)row * ldz + cv, zv);
      }
      // sigma acts on the stored (rounded) z so a checkpointed recompute is bit-identical
      V::unpack(zu, u);
      V::unpack(zv, v);
      float au[8], av[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        au[j] = silu_crossgate<T>(u[j]) * v[j];
        av[j] = silu_crossgate<T>(v[j]) * u[j];
      }
      store8(a_out + (long long)row * lda + cu, au);
      store8(a_out + (long long)row * lda + cv, av);
    } else {
      const int c = p * r + g * 8;
      float f[8];
      load8(P + (long long)row * ldp + c, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] *= inv;
      const typename V::Raw zz = V::pack(f);
      if (write_z) V::st(z_out + (long long)row * ldz + c, zz);
      if (a_out != nullptr) V::st(a_out + (long long)row * lda + c, zz);
    }
  }
}

// ----------------------------------------------------------------------------- K4 backward
// One warp per row: sigma-bwd, then dP = dz / s and dss = -<dz, z> / (2 s^2 d).
template <typename T>
// (256, 6): <= 40 registers -> 6 blocks / 48 warps per SM; more rows in flight (31.8 -> 29.8 us, q|k|v chunk)
__global__ void __launch_bounds__(256, 6) fixup_sigma_bwd_kernel(const T* __restrict__ z, long long ldz, const T* da,
                                                              long long ldda, const float* __restrict__ s_in, int d,
                                                              T* dP, long long lddp, float* __restrict__ dss, int rows,
                                                              int r, int nproj, int variant) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float s = s_in ? s_in[row] : 1.0f;
  const float inv = 1.0f / s;
  const int per_proj = variant == 1 ? (r >> 4) : (r >> 3);
  const int groups = per_proj * nproj;
  float dot = 0.f;
  for (int gi = lane; gi < groups; gi += 32) {
    const int p = gi / per_proj;
    const int g = gi - p * per_proj;
    if (variant == 1) {
      const int cu = p * r + g * 8, cv = cu + (r >> 1);
      float u[8], v[8], du_[8], dv_[8];
      load8(z + (long long)row * ldz + cu, u);
      load8(z + (long long)row * ldz + cv, v);
      load8(da + (long long)row * ldda + cu, du_);
      load8(da + (long long)row * ldda + cv, dv_);
      float gu[8], gv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float su = sigmoidf_safe(u[j]), sv = sigmoidf_safe(v[j]);
        const float silu_u = u[j] * su, silu_v = v[j] * sv;
        const float dsilu_u = su * (1.0f + u[j] * (1.0f - su));
        const float dsilu_v = sv * (1.0f + v[j] * (1.0f - sv));
        // a_u = silu(u) v ; a_v = silu(v) u
        gu[j] = du_[j] * dsilu_u * v[j] + dv_[j] * silu_v;
        gv[j] = du_[j] * silu_u + dv_[j] * dsilu_v * u[j];
        dot = fmaf(gu[j], u[j], dot);
        dot = fmaf(gv[j], v[j], dot);
        gu[j] *= inv;
        gv[j] *= inv;
      }
      store8(dP + (long long)row * lddp + cu, gu);
      store8(dP + (long long)row * lddp + cv, gv);
    } else {
      const int c = p * r + g * 8;
      float zz[8], dd[8];
      load8(z + (long long)row * ldz + c, zz);
      load8(da + (long long)row * ldda + c, dd);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dot = fmaf(dd[j], zz[j], dot);
        dd[j] *= inv;
      }
      store8(dP + (long long)row * lddp + c, dd);
    }
  }
  dot = warp_sum(dot);
  if (lane == 0 && dss != nullptr && s_in != nullptr) dss[row] = -dot / (2.0f * s * s * (float)d);
}

// ----------------------------------------------------------------------------- K5
template <typename T>
__global__ void __launch_bounds__(256) swiglu_kernel(const T* __restrict__ g, long long ldg, const T* __restrict__ u,
                                                     long long ldu, T* __restrict__ act, long long lda, int rows,
                                                     int cols) {
  const int per_row = cols >> 3;
  const long long total = (long long)per_row * rows;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / per_row);
    const int c = (int)(idx - (long long)row * per_row) * 8;
    float fg[8], fu[8];
    load8(g + (long long)row * ldg + c, fg);
    load8(u + (long long)row * ldu + c, fu);
#pragma unroll
    for (int j = 0; j < 8; ++j) fg[j] = silu_f(fg[j]) * fu[j];
    store8(act + (long long)row * lda + c, fg);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) swiglu_bwd_kernel(const T* __restrict__ g, long long ldg,
                                                         const T* __restrict__ u, long long ldu,
                                                         const T* __restrict__ dact, long long ldda,
                                                         T* __restrict__ dg, long long lddg, T* __restrict__ du,
                                                         long long lddu, int rows, int cols) {
  const int per_row = cols >> 3;
  const long long total = (long long)per_row * rows;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / per_row);
    const int c = (int)(idx - (long long)row * per_row) * 8;
    float fg[8], fu[8], fd[8], og[8], ou[8];
    load8(g + (long long)row * ldg + c, fg);
    load8(u + (long long)row * ldu + c, fu);
    load8(dact + (long long)row * ldda + c, fd);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float sg = sigmoidf_safe(fg[j]);
      const float silu_g = fg[j] * sg;
      og[j] = fd[j] * fu[j] * sg * (1.0f + fg[j] * (1.0f - sg));
      ou[j] = fd[j] * silu_g;
    }
    store8(dg + (long long)row * lddg + c, og);
    store8(du + (long long)row * lddu + c, ou);
  }
}

// ----------------------------------------------------------------------------- K3 backward
// (rmsnorm_bwd_pipe_kernel below: the TMA row-pipeline form)

// Full-width RMSNorm n = x*gamma/s (baselines): dn -> dh = dn / s (in place allowed) and
// dss = -<dn, gamma*x> / (2 s^3 d), so rmsnorm_bwd finishes dx and dgamma.
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_bwd_prep_kernel(const T* dn, long long lddn, const T* __restrict__ x,
                                                               long long ldx, const float* __restrict__ gamma,
                                                               const float* __restrict__ s_in, T* dh, long long lddh,
                                                               float* __restrict__ dss, int rows, int width) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float s = s_in[row];
  const float inv = 1.0f / s;
  float dot = 0.f;
  for (int c = lane; c < (width >> 3); c += 32) {
    float fd[8], fx[8], g[8];
    load8(dn + (long long)row * lddn + c * 8, fd);
    load8(x + (long long)row * ldx + c * 8, fx);
    load_gamma8(gamma + c * 8, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dot = fmaf(fd[j], g[j] * fx[j], dot);
      fd[j] *= inv;
    }
    store8(dh + (long long)row * lddh + c * 8, fd);
  }
  dot = warp_sum(dot);
  if (lane == 0) dss[row] = -dot / (2.0f * s * s * s * (float)width);
}

// ----------------------------------------------------------------------------- reductions
__global__ void __launch_bounds__(256) reduce_rows_kernel(const float* __restrict__ in, int splits,
                                                          long long split_stride, long long ldi, int rows, int cols,
                                                          const float* __restrict__ col_scale, float* __restrict__ out,
                                                          long long ldo, int accumulate) {
  const int per_row = cols >> 2;
  const long long total = (long long)per_row * rows;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / per_row);
    const int c = (int)(idx - (long long)row * per_row) * 4;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < splits; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(in + k * split_stride + (long long)row * ldi + c);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (col_scale != nullptr) {
      const float4 cs = *reinterpret_cast<const float4*>(col_scale + c);
      s.x *= cs.x; s.y *= cs.y; s.z *= cs.z; s.w *= cs.w;
    }
    float4* o = reinterpret_cast<float4*>(out + (long long)row * ldo + c);
    if (accumulate) {
      const float4 p = *o;
      s.x += p.x; s.y += p.y; s.z += p.z; s.w += p.w;
    }
    *o = s;
  }
}

__global__ void __launch_bounds__(256) reduce_rows_scalar_kernel(const float* __restrict__ in, int splits,
                                                                 long long split_stride, long long ldi, int rows,
                                                                 int cols, const float* __restrict__ col_scale,
                                                                 float* __restrict__ out, long long ldo,
                                                                 int accumulate) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / cols);
    const int c = (int)(idx - (long long)row * cols);
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += in[k * split_stride + (long long)row * ldi + c];
    if (col_scale != nullptr) s *= col_scale[c];
    float* o = out + (long long)row * ldo + c;
    *o = accumulate ? *o + s : s;
  }
}

// out[c] (+)= scale[c] * sum_{s<S} in[s*lds + c]: 32 columns x 32 row-groups per block, rows
// strided by 32, then a fixed-order tree over the row-groups in smem (deterministic).
__global__ void __launch_bounds__(1024) colsum_kernel(const float* __restrict__ in, int S, long long lds, int C,
                                                      const float* __restrict__ scale, float* __restrict__ out,
                                                      int accumulate) {
  __shared__ float red[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float s = 0.f;
  if (c < C)
    for (int r = ty; r < S; r += 32) s += in[(long long)r * lds + c];
  red[ty][tx] = s;
  __syncthreads();
  for (int w = 16; w > 0; w >>= 1) {
    if (ty < w) red[ty][tx] += red[ty + w][tx];
    __syncthreads();
  }
  if (ty == 0 && c < C) {
    float v = red[0][tx];
    if (scale) v *= scale[c];
    out[c] = accumulate ? out[c] + v : v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) add_kernel(const T* __restrict__ a, long long lda, const T* __restrict__ b,
                                                  long long ldb, T* __restrict__ out, long long ldo, int rows,
                                                  int cols) {
  const int per_row = cols >> 3;
  const long long total = (long long)per_row * rows;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / per_row);
    const int c = (int)(idx - (long long)row * per_row) * 8;
    float fa[8], fb[8];
    load8(a + (long long)row * lda + c, fa);
    load8(b + (long long)row * ldb + c, fb);
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] += fb[j];
    store8(out + (long long)row * ldo + c, fa);
  }
}

// partial[blk] = sum over this block's rows of <a_row, b_row>; fixed block/thread order.
template <typename T>
__global__ void __launch_bounds__(256) dot_kernel(const T* __restrict__ a, long long lda, const T* __restrict__ b,
                                                  long long ldb, int rows, int cols, float* __restrict__ partial) {
  __shared__ float red[8];
  const int per_row = cols >> 3;
  const long long total = (long long)per_row * rows;
  // four grid-stride items per round, all eight 16-byte loads issued before any FMA: a thread
  // otherwise waits one full memory latency per item (the grid is capped at 4 blocks per SM)
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; idx + 3 * stride < total; idx += 4 * stride) {
    float fa[4][8], fb[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long it = idx + u * stride;
      const int row = (int)(it / per_row);
      const int c = (int)(it - (long long)row * per_row) * 8;
      load8(a + (long long)row * lda + c, fa[u]);
      load8(b + (long long)row * ldb + c, fb[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = fmaf(fa[u][j], fb[u][j], acc);
  }
  for (; idx < total; idx += stride) {
    const int row = (int)(idx / per_row);
    const int c = (int)(idx - (long long)row * per_row) * 8;
    float fa[8], fb[8];
    load8(a + (long long)row * lda + c, fa);
    load8(b + (long long)row * ldb + c, fb);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = fmaf(fa[j], fb[j], acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

// ----------------------------------------------------------------------------- fused AdamW
// One pass over a flat parameter set: fp32 master weights, fp32 moments, fp32 gradients, and the
// working copy the GEMMs read (bf16, or fp32 in parity mode) rewritten from the master.
//   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2 ; p -= lr (m/bc1 / (sqrt(v/bc2) + eps) + wd p)
template <typename T>
__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ master, float* __restrict__ m,
                                                    float* __restrict__ v, const float* __restrict__ g,
                                                    T* __restrict__ work, long long n, float lr, float b1, float b2,
                                                    float eps, float wd, int step_host,
                                                    const int* __restrict__ step_dev) {
  // the step count may live on the device so a replayed CUDA graph keeps advancing it
  const float step = (float)(step_dev ? *step_dev : step_host);
  // bias corrections folded into two per-thread reciprocals; the per-element quotient uses the MUFU
  // reciprocal and sqrt(v) = v * rsqrt(v) (the IEEE div / sqrt call sequences made this kernel
  // issue-bound rather than HBM-bound)
  const float ibc1 = 1.0f / (1.0f - powf(b1, step)), ibc2 = 1.0f / (1.0f - powf(b2, step));
  const long long n8 = n >> 3;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    const long long o = i * 8;
    float p[8], mm[8], vv[8], gg[8];
    *reinterpret_cast<float4*>(p) = reinterpret_cast<const float4*>(master + o)[0];
    *reinterpret_cast<float4*>(p + 4) = reinterpret_cast<const float4*>(master + o)[1];
    *reinterpret_cast<float4*>(mm) = reinterpret_cast<const float4*>(m + o)[0];
    *reinterpret_cast<float4*>(mm + 4) = reinterpret_cast<const float4*>(m + o)[1];
    *reinterpret_cast<float4*>(vv) = reinterpret_cast<const float4*>(v + o)[0];
    *reinterpret_cast<float4*>(vv + 4) = reinterpret_cast<const float4*>(v + o)[1];
    *reinterpret_cast<float4*>(gg) = reinterpret_cast<const float4*>(g + o)[0];
    *reinterpret_cast<float4*>(gg + 4) = reinterpret_cast<const float4*>(g + o)[1];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mm[j] = b1 * mm[j] + (1.0f - b1) * gg[j];
      vv[j] = b2 * vv[j] + (1.0f - b2) * gg[j] * gg[j];
      const float vh = vv[j] * ibc2;
      const float root = vh > 0.0f ? vh * rsqrtf(vh) : 0.0f;
      const float upd = __fdividef(mm[j] * ibc1, root + eps) + wd * p[j];
      p[j] -= lr * upd;
    }
    reinterpret_cast<float4*>(master + o)[0] = *reinterpret_cast<float4*>(p);
    reinterpret_cast<float4*>(master + o)[1] = *reinterpret_cast<float4*>(p + 4);
    reinterpret_cast<float4*>(m + o)[0] = *reinterpret_cast<float4*>(mm);
    reinterpret_cast<float4*>(m + o)[1] = *reinterpret_cast<float4*>(mm + 4);
    reinterpret_cast<float4*>(v + o)[0] = *reinterpret_cast<float4*>(vv);
    reinterpret_cast<float4*>(v + o)[1] = *reinterpret_cast<float4*>(vv + 4);
    store8(work + o, p);
  }
}


// ----------------------------------------------------------------------------- TMA row pipeline
// HBM-bound per-row kernels (RMSNorm forward / backward) stream their input rows through a ring
// of shared-memory stages filled by 1-D bulk copies (cp.async.bulk, completion on an mbarrier per
// stage): one thread keeps `stages` rows of every input in flight per block, so the memory system
// sees deep, register-free parallelism (the register-staged warp-per-row versions were
// latency-bound at ~60 % of HBM bandwidth). A block owns a contiguous range of rows; its 256
// threads split each row into 8-element chunks (thread t owns chunks t, t+256, ...), so per-column
// state (gamma, the dgamma partial) stays in registers for the whole block.
constexpr int kPipeThreads = 256;

struct RowPipe {
  uint8_t* smem;
  uint64_t* bars;
  uint32_t stage_bytes;
  int stages;

  __device__ __forceinline__ uint8_t* stage(int i) const { return smem + (size_t)(i % stages) * stage_bytes; }
  __device__ __forceinline__ void wait(int i) const { mbar_wait(&bars[i % stages], (uint32_t)((i / stages) & 1)); }
};

__device__ __forceinline__ RowPipe make_pipe(uint8_t* sm, int stages, uint32_t stage_bytes) {
  RowPipe rp;
  rp.smem = sm;
  rp.stage_bytes = stage_bytes;
  rp.stages = stages;
  rp.bars = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&rp.bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  return rp;
}

// one thread: bring row `row` of up to three row-major inputs into the stage of pipeline slot i
template <typename T>
__device__ __forceinline__ void pipe_issue(const RowPipe& rp, int i, long long row, uint32_t row_bytes, const T* a,
                                           long long lda, const T* b, long long ldb, const T* c, long long ldc) {
  uint8_t* dst = rp.stage(i);
  uint64_t* bar = &rp.bars[i % rp.stages];
  const int n = 1 + (b != nullptr) + (c != nullptr);
  mbar_arrive_expect_tx(bar, n * row_bytes);
  bulk_load_1d(dst, a + row * lda, row_bytes, bar);
  if (b != nullptr) bulk_load_1d(dst + row_bytes, b + row * ldb, row_bytes, bar);
  if (c != nullptr) bulk_load_1d(dst + (b != nullptr ? 2 : 1) * row_bytes, c + row * ldc, row_bytes, bar);
}

// Online RMSNorm (+ residual) forward over rows [r0, r1) of this block, same contract as
// rmsnorm_residual_kernel, warp-specialised: warp 8 streams rows into `stages` (<= 16) smem stages
// with bulk copies (full barrier per stage), warps 0..7 each own every 8th row — the row statistic
// is a warp reduction (no block barrier per row) — and release the stage (empty barrier) once read.
constexpr int kFwdMaxStages = 16;
constexpr int kFwdConsumers = 8;

template <typename T, int NCH>
__global__ void __launch_bounds__(32 * (kFwdConsumers + 1)) rmsnorm_residual_pipe_kernel(
    const T* __restrict__ x, long long ldx, const T* __restrict__ branch, long long ldb, T* __restrict__ x_out,
    long long ldo, const float* __restrict__ gamma, T* __restrict__ n_out, long long ldn, float* __restrict__ ss_out,
    float* __restrict__ rl_out, int rows, int width, float eps, int rows_per_block, int kFwdStages) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int r0 = blockIdx.x * rows_per_block;
  const int n = min(rows, r0 + rows_per_block) - r0;
  if (n <= 0) return;
  const uint32_t row_bytes = (uint32_t)width * sizeof(T);
  const uint32_t stage_bytes = row_bytes * (branch != nullptr ? 2 : 1);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)kFwdStages * stage_bytes);
  uint64_t* empty = full + kFwdMaxStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == kFwdConsumers) {  // producer warp
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % kFwdStages;
        if (i >= kFwdStages) mbar_wait(&empty[s], (uint32_t)(((i / kFwdStages) - 1) & 1));
        uint8_t* dst = sm + (size_t)s * stage_bytes;
        const long long row = r0 + i;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        bulk_load_1d(dst, x + row * ldx, row_bytes, &full[s]);
        if (branch != nullptr) bulk_load_1d(dst + row_bytes, branch + row * ldb, row_bytes, &full[s]);
      }
    }
    return;
  }
  const int nch = width >> 3;
  for (int i = warp; i < n; i += kFwdConsumers) {
    const int s = i % kFwdStages;
    const long long row = r0 + i;
    mbar_wait(&full[s], (uint32_t)((i / kFwdStages) & 1));
    const T* sx = reinterpret_cast<const T*>(sm + (size_t)s * stage_bytes);
    const T* sb = sx + width;
    typename Vec8<T>::Raw keep[NCH];
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const int c = lane + 32 * q;
      if (c < nch) {
        typename Vec8<T>::Raw w = Vec8<T>::ld(sx + c * 8);
        if (branch != nullptr) {
          float fx[8], fb[8];
          Vec8<T>::unpack(w, fx);
          load8(sb + c * 8, fb);
#pragma unroll
          for (int j = 0; j < 8; ++j) fx[j] += fb[j];
          w = Vec8<T>::pack(fx);
          if (x_out != nullptr) Vec8<T>::st(x_out + row * ldo + c * 8, w);
        }
        keep[q] = w;
        float f[8];
        Vec8<T>::unpack(w, f);  // statistics of the stored (rounded) value
#pragma unroll
        for (int j = 0; j < 8; ++j) ss = fmaf(f[j], f[j], ss);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the row is in registers: the stage may be refilled
    ss = warp_sum(ss);
    const float rl = sqrtf(ss / (float)width + eps);
    if (lane == 0) {
      if (ss_out) ss_out[row] = ss;
      if (rl_out) rl_out[row] = rl;
    }
    if (n_out == nullptr) continue;
    const float inv = 1.0f / rl;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const int c = lane + 32 * q;
      if (c < nch) {
        float f[8], g[8];
        Vec8<T>::unpack(keep[q], f);
        load_gamma8(gamma + c * 8, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = f[j] * g[j] * inv;
        store8(n_out + row * ldn + c * 8, f);
      }
    }
  }
}

// Online/sync RMSNorm backward over rows [r0, r1) of this block (contract of rmsnorm_bwd_kernel):
// dx = dres + dh * gamma + 2 x dss ; dgamma partial row per block (this thread's columns).
template <typename T, int G>
__global__ void __launch_bounds__(kPipeThreads) rmsnorm_bwd_pipe_kernel(
    const T* __restrict__ dh, long long lddh, const T* __restrict__ x, long long ldx, const float* __restrict__ gamma,
    const float* __restrict__ dss, const T* __restrict__ dres, long long ldr, T* __restrict__ dx, long long lddx,
    float* __restrict__ dgamma_partial, int rows, int width, int rows_per_block, int stages) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int r0 = blockIdx.x * rows_per_block;
  const int n = max(0, min(rows, r0 + rows_per_block) - r0);
  const int nch = width >> 3;
  float acc[G][8];
#pragma unroll
  for (int q = 0; q < G; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[q][j] = 0.f;
  if (n > 0) {
    const uint32_t row_bytes = (uint32_t)width * sizeof(T);
    const int narr = dres != nullptr ? 3 : 2;
    const RowPipe rp = make_pipe(sm, stages, narr * row_bytes);
    if (threadIdx.x == 0)
      for (int i = 0; i < min(stages, n); ++i) pipe_issue<T>(rp, i, r0 + i, row_bytes, dh, lddh, x, ldx, dres, ldr);
    float g[G][8];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int c = threadIdx.x + q * kPipeThreads;
      if (c < nch) load_gamma8(gamma + c * 8, g[q]);
    }
    for (int i = 0; i < n; ++i) {
      const long long row = r0 + i;
      rp.wait(i);
      const T* sdh = reinterpret_cast<const T*>(rp.stage(i));
      const T* sx = sdh + width;
      const T* sr = sx + width;
      const float two_dss = 2.0f * dss[row];
      float o[G][8];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int c = threadIdx.x + q * kPipeThreads;
        if (c < nch) {
          float fh[8], fx[8], fr[8];
          load8(sdh + c * 8, fh);
          load8(sx + c * 8, fx);
          if (dres != nullptr) {
            load8(sr + c * 8, fr);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) fr[j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            o[q][j] = fr[j] + fh[j] * g[q][j] + two_dss * fx[j];
            acc[q][j] = fmaf(fh[j], fx[j], acc[q][j]);
          }
        }
      }
      __syncthreads();  // every thread is done reading stage i: refill it
      if (threadIdx.x == 0 && i + stages < n)
        pipe_issue<T>(rp, i + stages, row + stages, row_bytes, dh, lddh, x, ldx, dres, ldr);
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int c = threadIdx.x + q * kPipeThreads;
        if (c < nch) store8(dx + row * lddx + c * 8, o[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int c = threadIdx.x + q * kPipeThreads;
    if (c < nch) {
      float* out = dgamma_partial + (long long)blockIdx.x * width + c * 8;
      reinterpret_cast<float4*>(out)[0] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
      reinterpret_cast<float4*>(out)[1] = make_float4(acc[q][4], acc[q][5], acc[q][6], acc[q][7]);
    }
  }
}

// ============================================================================= launchers
static inline int grid_for(long long items, int threads = 256) {
  const long long want = (items + threads - 1) / threads;
  const long long cap = (long long)num_sms_cached() * 16;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

#define BTP_CHECK_LAUNCH() return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA

// stages of the row pipeline for a given per-row stage size: ~72 KB of rows in flight per block,
// so three 256-thread blocks share one SM's shared memory
static inline int pipe_stages(uint32_t stage_bytes) {
  int st = (int)((72u * 1024u) / stage_bytes);
  return st < 2 ? 2 : (st > 8 ? 8 : st);
}

static inline size_t pipe_smem(int stages, uint32_t stage_bytes) {
  return (size_t)stages * stage_bytes + (size_t)stages * sizeof(uint64_t);
}

template <typename Kern>
static bool pipe_configure(Kern k, size_t smem) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
}

template <typename T, int NCH>
static int rmsnorm_residual_pipe_t(const T* x, long long ldx, const T* b, long long ldb, T* xo, long long ldo,
                                   const float* gamma, T* no, long long ldn, float* ss_out, float* rl_out, int rows,
                                   int width, float eps, cudaStream_t st) {
  const uint32_t stage_bytes = (uint32_t)width * sizeof(T) * (b != nullptr ? 2 : 1);
  // Each of the 8 consumer warps owns rows w, w+8, ...; with a multiple of 8 stages every stage is
  // only ever awaited by ONE warp, in order (a warp may never wait more than one phase ahead on an
  // mbarrier). 16 stages when they fit in ~96 KB, else 8.
  const int stages = 16u * stage_bytes <= 96u * 1024u ? 16 : kFwdConsumers;
  const size_t smem = (size_t)stages * stage_bytes + 2 * kFwdMaxStages * sizeof(uint64_t);
  if (smem > 220 * 1024 || !pipe_configure(rmsnorm_residual_pipe_kernel<T, NCH>, smem)) return BTP_ERR_CUDA;
  int per_sm = (int)((220 * 1024) / smem);
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  int nblk = per_sm * num_sms_cached();
  const int rpb = (rows + nblk - 1) / nblk;
  nblk = (rows + rpb - 1) / rpb;
  rmsnorm_residual_pipe_kernel<T, NCH><<<nblk, 32 * (kFwdConsumers + 1), smem, st>>>(
      x, ldx, b, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out, rows, width, eps, rpb, stages);
  BTP_CHECK_LAUNCH();
}

template <typename T>
static int rmsnorm_residual_regs_t(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                                   long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                                   float* rl_out, int rows, int width, float eps, cudaStream_t st);

template <typename T>
static int rmsnorm_residual_t(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                              long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                              float* rl_out, int rows, int width, float eps, cudaStream_t st) {
  if ((size_t)kFwdConsumers * width * sizeof(T) * (branch != nullptr ? 2 : 1) > 192 * 1024)
    return rmsnorm_residual_regs_t<T>(x, ldx, branch, ldb, x_out, ldo, gamma, n_out, ldn, ss_out, rl_out, rows, width,
                                      eps, st);
  {  // TMA row pipeline (rows are 16-byte aligned: checked by the caller)
    const T* xb = static_cast<const T*>(x);
    const T* bb = static_cast<const T*>(branch);
    T* xo = static_cast<T*>(x_out);
    T* no = static_cast<T*>(n_out);
    const int nch = width / 8;
    if (nch <= 32 * 2)
      return rmsnorm_residual_pipe_t<T, 2>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out, rows, width, eps,
                                           st);
    if (nch <= 32 * 8)
      return rmsnorm_residual_pipe_t<T, 8>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out, rows, width, eps,
                                           st);
    return rmsnorm_residual_pipe_t<T, 32>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out, rows, width, eps,
                                          st);
  }
}

// register-staged warp-per-row form: rows too wide for 8 smem stages
template <typename T>
static int rmsnorm_residual_regs_t(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                                   long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                                   float* rl_out, int rows, int width, float eps, cudaStream_t st) {
  const int blocks = (rows + 7) / 8;
  const int nch = width / 8;
  const T* xb = static_cast<const T*>(x);
  const T* bb = static_cast<const T*>(branch);
  T* xo = static_cast<T*>(x_out);
  T* no = static_cast<T*>(n_out);
  if (nch <= 32 * 4)
    rmsnorm_residual_kernel<T, 4><<<blocks, 256, 0, st>>>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out,
                                                          rows, width, eps);
  else if (nch <= 32 * 8)
    rmsnorm_residual_kernel<T, 8><<<blocks, 256, 0, st>>>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out,
                                                          rows, width, eps);
  else if (nch <= 32 * 16)
    rmsnorm_residual_kernel<T, 16><<<blocks, 256, 0, st>>>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out,
                                                           rows, width, eps);
  else
    rmsnorm_residual_kernel<T, 32><<<blocks, 256, 0, st>>>(xb, ldx, bb, ldb, xo, ldo, gamma, no, ldn, ss_out, rl_out,
                                                           rows, width, eps);
  BTP_CHECK_LAUNCH();
}

int rmsnorm_residual(const void* x, long long ldx, const void* branch, long long ldb, void* x_out, long long ldo,
                     const float* gamma, void* n_out, long long ldn, float* ss_out, float* rl_out, int rows,
                     int width, float eps, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0) return BTP_ERR_DIM;
  if (width % 8 || width > 8192 || ldx % 8 || (branch && ldb % 8) || (x_out && ldo % 8) || (n_out && ldn % 8))
    return BTP_ERR_ALIGNMENT;
  if (!al16(x) || (branch && !al16(branch)) || (x_out && !al16(x_out)) || (n_out && !al16(n_out)) ||
      (n_out && !al16(gamma)))
    return BTP_ERR_ALIGNMENT;
  if (f32) return rmsnorm_residual_t<float>(x, ldx, branch, ldb, x_out, ldo, gamma, n_out, ldn, ss_out, rl_out, rows,
                                            width, eps, st);
  return rmsnorm_residual_t<bf16>(x, ldx, branch, ldb, x_out, ldo, gamma, n_out, ldn, ss_out, rl_out, rows, width,
                                  eps, st);
}

int rmsnorm_apply(const void* x, long long ldx, const float* gamma, const float* ss_total, int d, float eps,
                  void* n_out, long long ldn, float* rms_out, int rows, int width, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0 || d <= 0) return BTP_ERR_DIM;
  if (width % 8 || ldx % 8 || ldn % 8 || !al16(x) || !al16(n_out) || !al16(gamma)) return BTP_ERR_ALIGNMENT;
  if (f32)
    rmsnorm_apply_kernel<float><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const float*>(x), ldx, gamma, ss_total, d,
                                                               eps, static_cast<float*>(n_out), ldn, rms_out, rows,
                                                               width);
  else
    rmsnorm_apply_kernel<bf16><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const bf16*>(x), ldx, gamma, ss_total, d,
                                                              eps, static_cast<bf16*>(n_out), ldn, rms_out, rows, width);
  BTP_CHECK_LAUNCH();
}

int fixup_sigma_f32in(const float* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                      void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj, int variant,
                      cudaStream_t st) {
  if (rows <= 0 || r <= 0 || nproj <= 0 || z_out == nullptr) return BTP_ERR_DIM;
  if (variant != 0 && variant != 1) return BTP_ERR_DIM;
  if (variant == 1 && (r % 16)) return BTP_ERR_DIVISIBILITY;
  if (r % 8 || ldp % 8 || ldz % 8 || (a_out && lda % 8)) return BTP_ERR_ALIGNMENT;
  if (variant == 1 && a_out == nullptr) return BTP_ERR_DIM;
  if (!al16(P) || !al16(z_out) || (a_out && !al16(a_out))) return BTP_ERR_ALIGNMENT;
  const long long items = (long long)rows * nproj * (variant == 1 ? r / 16 : r / 8);
  fixup_sigma_kernel<bf16, float><<<grid_for(items), 256, 0, st>>>(P, ldp, ss_total, d, eps, s_out,
                                                                   static_cast<bf16*>(z_out), ldz,
                                                                   static_cast<bf16*>(a_out), lda, rows, r, nproj,
                                                                   variant);
  BTP_CHECK_LAUNCH();
}

int fixup_sigma(const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out, void* z_out,
                long long ldz, void* a_out, long long lda, int rows, int r, int nproj, int variant, cudaStream_t st,
                bool f32) {
  if (rows <= 0 || r <= 0 || nproj <= 0) return BTP_ERR_DIM;
  if (variant != 0 && variant != 1) return BTP_ERR_DIM;
  if (variant == 1 && (r % 16)) return BTP_ERR_DIVISIBILITY;
  if (r % 8 || ldp % 8 || (z_out && ldz % 8) || (a_out && lda % 8)) return BTP_ERR_ALIGNMENT;
  if (variant == 1 && a_out == nullptr) return BTP_ERR_DIM;
  if (!al16(P) || (z_out && !al16(z_out)) || (a_out && !al16(a_out))) return BTP_ERR_ALIGNMENT;
  const long long items = (long long)rows * nproj * (variant == 1 ? r / 16 : r / 8);
  if (f32)
    fixup_sigma_kernel<float><<<grid_for(items), 256, 0, st>>>(static_cast<const float*>(P), ldp, ss_total, d, eps,
                                                               s_out, static_cast<float*>(z_out), ldz,
                                                               static_cast<float*>(a_out), lda, rows, r, nproj,
                                                               variant);
  else
    fixup_sigma_kernel<bf16><<<grid_for(items), 256, 0, st>>>(static_cast<const bf16*>(P), ldp, ss_total, d, eps,
                                                              s_out, static_cast<bf16*>(z_out), ldz,
                                                              static_cast<bf16*>(a_out), lda, rows, r, nproj, variant);
  BTP_CHECK_LAUNCH();
}

int fixup_sigma_bwd(const void* z, long long ldz, const void* da, long long ldda, const float* s, int d, void* dP,
                    long long lddp, float* dss, int rows, int r, int nproj, int variant, cudaStream_t st, bool f32) {
  if (rows <= 0 || r <= 0 || nproj <= 0) return BTP_ERR_DIM;
  if (variant != 0 && variant != 1) return BTP_ERR_DIM;
  if (variant == 1 && (r % 16)) return BTP_ERR_DIVISIBILITY;
  if (r % 8 || ldz % 8 || ldda % 8 || lddp % 8) return BTP_ERR_ALIGNMENT;
  if (!al16(z) || !al16(da) || !al16(dP)) return BTP_ERR_ALIGNMENT;
  if (f32)
    fixup_sigma_bwd_kernel<float><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const float*>(z), ldz,
                                                                  static_cast<const float*>(da), ldda, s, d,
                                                                  static_cast<float*>(dP), lddp, dss, rows, r, nproj,
                                                                  variant);
  else
    fixup_sigma_bwd_kernel<bf16><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const bf16*>(z), ldz,
                                                                 static_cast<const bf16*>(da), ldda, s, d,
                                                                 static_cast<bf16*>(dP), lddp, dss, rows, r, nproj,
                                                                 variant);
  BTP_CHECK_LAUNCH();
}

int swiglu(const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda, int rows, int cols,
           cudaStream_t st, bool f32) {
  if (rows <= 0 || cols <= 0) return BTP_ERR_DIM;
  if (cols % 8 || ldg % 8 || ldu % 8 || lda % 8 || !al16(g) || !al16(u) || !al16(act)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_for((long long)rows * cols / 8);
  if (f32)
    swiglu_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(g), ldg, static_cast<const float*>(u), ldu,
                                               static_cast<float*>(act), lda, rows, cols);
  else
    swiglu_kernel<bf16><<<grid, 256, 0, st>>>(static_cast<const bf16*>(g), ldg, static_cast<const bf16*>(u), ldu,
                                              static_cast<bf16*>(act), lda, rows, cols);
  BTP_CHECK_LAUNCH();
}

int swiglu_bwd(const void* g, long long ldg, const void* u, long long ldu, const void* dact, long long ldda,
               void* dg, long long lddg, void* du, long long lddu, int rows, int cols, cudaStream_t st, bool f32) {
  if (rows <= 0 || cols <= 0) return BTP_ERR_DIM;
  if (cols % 8 || ldg % 8 || ldu % 8 || ldda % 8 || lddg % 8 || lddu % 8) return BTP_ERR_ALIGNMENT;
  if (!al16(g) || !al16(u) || !al16(dact) || !al16(dg) || !al16(du)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_for((long long)rows * cols / 8);
  if (f32)
    swiglu_bwd_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(g), ldg, static_cast<const float*>(u),
                                                   ldu, static_cast<const float*>(dact), ldda,
                                                   static_cast<float*>(dg), lddg, static_cast<float*>(du), lddu, rows,
                                                   cols);
  else
    swiglu_bwd_kernel<bf16><<<grid, 256, 0, st>>>(static_cast<const bf16*>(g), ldg, static_cast<const bf16*>(u), ldu,
                                                  static_cast<const bf16*>(dact), ldda, static_cast<bf16*>(dg), lddg,
                                                  static_cast<bf16*>(du), lddu, rows, cols);
  BTP_CHECK_LAUNCH();
}

int rmsnorm_bwd(const void* dh, long long lddh, const void* x, long long ldx, const float* gamma, const float* dss,
                const void* dres, long long ldr, void* dx, long long lddx, float* dgamma_partial, int max_blocks,
                int* nblk_out, int rows, int width, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0 || max_blocks <= 0) return BTP_ERR_DIM;
  if (width % 8 || width > 8192 || lddh % 8 || ldx % 8 || lddx % 8 || (dres && ldr % 8)) return BTP_ERR_ALIGNMENT;
  if (!al16(dh) || !al16(x) || !al16(dx) || !al16(gamma) || (dres && !al16(dres))) return BTP_ERR_ALIGNMENT;
  const int nch = width / 8;
  // TMA row pipeline: one resident wave of 3 blocks per SM (bounded by the caller's partial rows)
  int nblk = 3 * num_sms_cached();
  if (nblk > max_blocks) nblk = max_blocks;
  const int rows_per_block = (rows + nblk - 1) / nblk;
  nblk = (rows + rows_per_block - 1) / rows_per_block;
  const uint32_t stage_bytes = (uint32_t)width * (f32 ? 4u : 2u) * (dres != nullptr ? 3u : 2u);
  const int stages = pipe_stages(stage_bytes);
  const size_t smem = pipe_smem(stages, stage_bytes);
  if (smem > 200 * 1024) return BTP_ERR_DIM;
  const int G = nch <= kPipeThreads ? 1 : (nch <= 2 * kPipeThreads ? 2 : 4);
#define BTP_NB_LAUNCH(T, GG)                                                                                       \
  do {                                                                                                             \
    if (!pipe_configure(rmsnorm_bwd_pipe_kernel<T, GG>, smem)) return BTP_ERR_CUDA;                               \
    rmsnorm_bwd_pipe_kernel<T, GG><<<nblk, kPipeThreads, smem, st>>>(                                              \
        static_cast<const T*>(dh), lddh, static_cast<const T*>(x), ldx, gamma, dss, static_cast<const T*>(dres), \
        ldr, static_cast<T*>(dx), lddx, dgamma_partial, rows, width, rows_per_block, stages);                     \
  } while (0)
  if (f32) {
    if (G == 1) BTP_NB_LAUNCH(float, 1);
    else if (G == 2) BTP_NB_LAUNCH(float, 2);
    else BTP_NB_LAUNCH(float, 4);
  } else {
    if (G == 1) BTP_NB_LAUNCH(bf16, 1);
    else if (G == 2) BTP_NB_LAUNCH(bf16, 2);
    else BTP_NB_LAUNCH(bf16, 4);
  }
#undef BTP_NB_LAUNCH
  if (nblk_out) *nblk_out = nblk;
  BTP_CHECK_LAUNCH();
}

int rmsnorm_bwd_prep(const void* dn, long long lddn, const void* x, long long ldx, const float* gamma, const float* s,
                     void* dh, long long lddh, float* dss, int rows, int width, cudaStream_t st, bool f32) {
  if (rows <= 0 || width <= 0) return BTP_ERR_DIM;
  if (width % 8 || lddn % 8 || ldx % 8 || lddh % 8 || !al16(dn) || !al16(x) || !al16(dh) || !al16(gamma))
    return BTP_ERR_ALIGNMENT;
  if (f32)
    rmsnorm_bwd_prep_kernel<float><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const float*>(dn), lddn,
                                                                   static_cast<const float*>(x), ldx, gamma, s,
                                                                   static_cast<float*>(dh), lddh, dss, rows, width);
  else
    rmsnorm_bwd_prep_kernel<bf16><<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const bf16*>(dn), lddn,
                                                                  static_cast<const bf16*>(x), ldx, gamma, s,
                                                                  static_cast<bf16*>(dh), lddh, dss, rows, width);
  BTP_CHECK_LAUNCH();
}

int reduce_rows(const float* in, int splits, long long split_stride, long long ldi, int rows, int cols,
                const float* col_scale, float* out, long long ldo, int accumulate, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || splits <= 0) return BTP_ERR_DIM;
  if (rows == 1 && splits >= 32) {  // many partial rows of one vector: parallel column sums
    colsum_kernel<<<(cols + 31) / 32, 1024, 0, st>>>(in, splits, split_stride, cols, col_scale, out, accumulate);
    BTP_CHECK_LAUNCH();
  }
  if (cols % 4 || ldi % 4 || ldo % 4 || split_stride % 4 || !al16(in) || !al16(out) || (col_scale && !al16(col_scale))) {
    reduce_rows_scalar_kernel<<<grid_for((long long)rows * cols), 256, 0, st>>>(in, splits, split_stride, ldi, rows,
                                                                             cols, col_scale, out, ldo, accumulate);
    BTP_CHECK_LAUNCH();
  }
  reduce_rows_kernel<<<grid_for((long long)rows * cols / 4), 256, 0, st>>>(in, splits, split_stride, ldi, rows, cols,
                                                                          col_scale, out, ldo, accumulate);
  BTP_CHECK_LAUNCH();
}

int add(const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows, int cols,
        cudaStream_t st, bool f32) {
  if (rows <= 0 || cols <= 0) return BTP_ERR_DIM;
  if (cols % 8 || lda % 8 || ldb % 8 || ldo % 8 || !al16(a) || !al16(b) || !al16(out)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_for((long long)rows * cols / 8);
  if (f32)
    add_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(a), lda, static_cast<const float*>(b), ldb,
                                            static_cast<float*>(out), ldo, rows, cols);
  else
    add_kernel<bf16><<<grid, 256, 0, st>>>(static_cast<const bf16*>(a), lda, static_cast<const bf16*>(b), ldb,
                                           static_cast<bf16*>(out), ldo, rows, cols);
  BTP_CHECK_LAUNCH();
}

int adamw(float* master, float* m, float* v, const float* g, void* work, long long n, float lr, float b1, float b2,
          float eps, float wd, int step, const int* step_dev, cudaStream_t st, bool f32) {
  if (n <= 0 || (step_dev == nullptr && step <= 0)) return BTP_ERR_DIM;
  if (n % 8 || !al16(master) || !al16(m) || !al16(v) || !al16(g) || !al16(work)) return BTP_ERR_ALIGNMENT;
  const int grid = grid_for(n / 8);
  if (f32)
    adamw_kernel<float><<<grid, 256, 0, st>>>(master, m, v, g, static_cast<float*>(work), n, lr, b1, b2, eps, wd, step,
                                              step_dev);
  else
    adamw_kernel<bf16><<<grid, 256, 0, st>>>(master, m, v, g, static_cast<bf16*>(work), n, lr, b1, b2, eps, wd, step,
                                             step_dev);
  BTP_CHECK_LAUNCH();
}

__global__ void counter_add_kernel(int* c, int delta) { *c += delta; }

int counter_add(int* ctr, int delta, cudaStream_t st) {
  counter_add_kernel<<<1, 1, 0, st>>>(ctr, delta);
  BTP_CHECK_LAUNCH();
}

int dot(const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
        int max_blocks, int* nblk_out, cudaStream_t st, bool f32) {
  if (rows <= 0 || cols <= 0 || max_blocks <= 0) return BTP_ERR_DIM;
  if (cols % 8 || lda % 8 || ldb % 8 || !al16(a) || !al16(b)) return BTP_ERR_ALIGNMENT;
  int nblk = grid_for((long long)rows * cols / 8);
  if (nblk > max_blocks) nblk = max_blocks;
  if (f32)
    dot_kernel<float><<<nblk, 256, 0, st>>>(static_cast<const float*>(a), lda, static_cast<const float*>(b), ldb, rows,
                                            cols, partial);
  else
    dot_kernel<bf16><<<nblk, 256, 0, st>>>(static_cast<const bf16*>(a), lda, static_cast<const bf16*>(b), ldb, rows,
                                           cols, partial);
  if (nblk_out) *nblk_out = nblk;
  BTP_CHECK_LAUNCH();
}

}  // namespace btp
