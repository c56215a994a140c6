// fp32 parity-mode GEMM: SIMT FFMA with fp32 accumulation (no TF32 rounding), same problem
// descriptor as the tcgen05 path (operand majors, row/col scale, residual, reduce-add).
//
// The north_star's fp32 tolerance (1e-4 relative vs the float64 reference) rules out
// single-pass TF32 (SURVEY §7 hard part 11); this kernel is the exact-fp32 CUDA path used when
// the block runs in fp32 mode. It is a correctness path, not the throughput path: 64x64 output
// tile per 256-thread block, 4x4 per thread, K staged through shared memory in steps of 16.
#include <cuda_runtime.h>

#include "btp_internal.h"

namespace btp {

constexpr int kTM = 64, kTN = 64, kTK = 16;

__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, long long lda, int a_mn,
                                                       const float* __restrict__ B, long long ldb, int b_mn,
                                                       float* C, long long ldc, int M, int N, int K,
                                                       const float* __restrict__ row_scale,
                                                       const float* __restrict__ col_scale, const float* resid,
                                                       long long ld_resid, float alpha, int reduce_add) {
  __shared__ float sA[kTK][kTM + 1];
  __shared__ float sB[kTK][kTN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * kTN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kTK) {
    for (int i = threadIdx.x; i < kTM * kTK; i += 256) {
      const int mm = i % kTM, kk = i / kTM;
      const int m = m0 + mm, k = k0 + kk;
      float va = 0.f, vb = 0.f;
      if (m < M && k < K) va = a_mn ? A[(long long)k * lda + m] : A[(long long)m * lda + k];
      sA[kk][mm] = va;
      const int n = n0 + mm;
      if (n < N && k < K) vb = b_mn ? B[(long long)k * ldb + n] : B[(long long)n * ldb + k];
      sB[kk][mm] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    const float rs = alpha * (row_scale ? row_scale[m] : 1.0f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] * rs;
      if (col_scale) v *= col_scale[n];
      if (resid) v += resid[(long long)m * ld_resid + n];
      float* c = C + (long long)m * ldc + n;
      *c = reduce_add ? *c + v : v;
    }
  }
}

int gemm_f32_launch(const btp_gemm_problem* probs, int n, cudaStream_t stream) {
  if (n <= 0 || n > 4) return BTP_ERR_DIM;
  for (int i = 0; i < n; ++i) {
    const btp_gemm_problem& q = probs[i];
    if (q.M <= 0 || q.N <= 0 || q.K <= 0) return BTP_ERR_DIM;
    if (!q.c_fp32 || q.epilogue != 0) return BTP_ERR_DIM;
    dim3 grid((q.N + kTN - 1) / kTN, (q.M + kTM - 1) / kTM);
    gemm_f32_kernel<<<grid, 256, 0, stream>>>(
        static_cast<const float*>(q.a), q.lda, q.a_mn, static_cast<const float*>(q.b), q.ldb, q.b_mn,
        static_cast<float*>(q.c), q.ldc, q.M, q.N, q.K, q.row_scale, q.col_scale, static_cast<const float*>(q.resid),
        q.ld_resid, q.alpha == 0.0f ? 1.0f : q.alpha, (q.reduce_add || q.splits > 1) ? 1 : 0);
    if (cudaGetLastError() != cudaSuccess) return BTP_ERR_CUDA;
  }
  return BTP_OK;
}

}  // namespace btp
