// Throughput of the forward softmax's exp2 loop (per element pair: FFMA2 scale, 2 x MUFU.EX2, FADD2
// row sum, F2FP bf16 pack; 128 scores held in registers per thread) at 1 / 2 / 4 warps per
// scheduler, one CTA per SM. Prints cycles per 128-score row-tile per warp and exp2 / clk / SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_12131_b200/csrc softmax_rate.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace btp;

constexpr int kReps = 256;

template <int kPoly, int kMode>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, long long* cyc, float seed) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = seed * (threadIdx.x + 3 * i) - 4.f;
  float l = 0.f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < kReps; ++r) {
    float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
    const float m = l * 1e-30f;
    const float2 c2 = make_float2(1.3f, 1.3f), nm = make_float2(-m, -m);
    if (kMode == 1) {
      // two phases: every exp2 first (MUFU back to back, results in place), then sums and packs
      float e[128];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), c2, nm);
        float2 y;
        if (kPoly > 0 && (i % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
          y = ex2_poly2(x);
        } else {
          y.x = ex2_approx(x.x);
          y.y = ex2_approx(x.y);
        }
        e[2 * i] = y.x;
        e[2 * i + 1] = y.y;
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 y = make_float2(e[2 * i], e[2 * i + 1]);
        if (i & 1) l2b = fadd2(l2b, y);
        else l2a = fadd2(l2a, y);
        acc ^= pack_bf16(y.x, y.y);
      }
      l += (l2a.x + l2a.y) + (l2b.x + l2b.y);
      continue;
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), c2, nm);
      float2 e;
      if (kPoly > 0 && (i % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
        e = ex2_poly2(x);
      } else {
        e.x = ex2_approx(x.x);
        e.y = ex2_approx(x.y);
      }
      if (i & 1) l2b = fadd2(l2b, e);
      else l2a = fadd2(l2a, e);
      acc ^= pack_bf16(e.x, e.y);
    }
    l += (l2a.x + l2a.y) + (l2b.x + l2b.y);
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(l);
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 16 + threadIdx.x / 32] = t1 - t0;
}

template <int kPoly, int kMode = 0>
void run(int warps, int nsm, uint32_t* out, long long* cyc) {
  k<kPoly, kMode><<<nsm, warps * 32>>>(out, cyc, 1e-3f);
  k<kPoly, kMode><<<nsm, warps * 32>>>(out, cyc, 1e-3f);
  cudaDeviceSynchronize();
  static long long h[148 * 16];
  cudaMemcpy(h, cyc, nsm * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < nsm; ++b)
    for (int w = 0; w < warps; ++w) mx = h[b * 16 + w] > mx ? h[b * 16 + w] : mx;
  const double per_tile = double(mx) / kReps;
  const double ex2_on_mufu = 128.0 * (kPoly > 0 ? 1.0 - 1.0 / kPoly : 1.0);
  printf("mode %d poly %d, %2d warps/CTA (%d per scheduler): %7.1f clk per 128-score tile per warp, %5.2f MUFU ex2/clk/SM, "
         "%5.2f exp2/clk/SM\n",
         kMode, kPoly, warps, warps / 4, per_tile, warps * 32 * ex2_on_mufu / per_tile, warps * 32 * 128.0 / per_tile);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, nsm * 512 * 4);
  cudaMalloc(&cyc, nsm * 16 * 8);
  for (int w : {4, 8, 16}) {
    run<0>(w, nsm, out, cyc);
    run<4>(w, nsm, out, cyc);
    run<0, 1>(w, nsm, out, cyc);
    run<4, 1>(w, nsm, out, cyc);
    run<3, 1>(w, nsm, out, cyc);
  }
  return 0;
}
