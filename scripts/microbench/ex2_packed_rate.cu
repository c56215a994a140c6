// MUFU exp2 throughput: ex2.approx.ftz.f32 vs the packed half forms (ex2.approx.f16x2,
// ex2.approx.ftz.bf16x2: two results per instruction), one 1024-thread CTA per SM, 8 independent
// chains per thread. Prints results (not instructions) per clk per SM, and the full softmax
// pair sequence built on f16x2 (FFMA2 scale, cvt to f16x2, MUFU, unpack, FADD2 row sum, bf16x2 pack).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_12131_b200/csrc ex2_packed_rate.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace btp;

#define N_IT 2048

__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int OP>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, long long* cyc, float seed) {
  float v[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) {
    v[i] = -seed * (threadIdx.x + i);
    u[i] = 0xbc00bc00u + i;  // f16x2 / bf16x2 small negatives
  }
  float2 acc = make_float2(0.f, 0.f);
  uint32_t pk = 0;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 1) u[i] = ex2_f16x2(u[i]) ^ 0x80008000u;
      if (OP == 2) u[i] = ex2_bf16x2(u[i]) ^ 0x80008000u;
      if (OP == 3) {  // softmax pair on f16x2: x = s c - m (FFMA2), cvt, MUFU, unpack, sum, bf16 pack
        const float2 x = ffma2(make_float2(v[i], v[(i + 1) & 7]), make_float2(1.3f, 1.3f), make_float2(-0.5f, -0.5f));
        uint32_t h;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x.y), "f"(x.x));
        const uint32_t e = ex2_f16x2(h);
        float lo, hi;
        asm("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\tcvt.f32.f16 %0, a;\n\tcvt.f32.f16 %1, b;\n\t}"
            : "=f"(lo), "=f"(hi) : "r"(e));
        acc = fadd2(acc, make_float2(lo, hi));
        pk ^= pack_bf16(lo, hi);
        v[i] += 1e-7f;
      }
    }
  }
  const long long t1 = clock64();
  uint32_t r = pk ^ __float_as_uint(acc.x + acc.y);
  for (int i = 0; i < 8; ++i) r ^= u[i] ^ __float_as_uint(v[i]);
  out[blockIdx.x * 1024 + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_instr, int nsm, uint32_t* out, long long* cyc) {
  k<OP><<<nsm, 1024>>>(out, cyc, 1e-3f);
  k<OP><<<nsm, 1024>>>(out, cyc, 1e-3f);
  cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = 1024.0 * N_IT * 8;
  printf("%-44s %6.1f instr / clk / SM  %6.1f exp2 results / clk / SM\n", name, ops / mx, per_instr * ops / mx);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, nsm * 1024 * 4);
  cudaMalloc(&cyc, nsm * 8);
  run<0>("ex2.approx.ftz.f32", 1, nsm, out, cyc);
  run<1>("ex2.approx.f16x2", 2, nsm, out, cyc);
  run<2>("ex2.approx.ftz.bf16x2", 2, nsm, out, cyc);
  run<3>("softmax pair via f16x2 (per pair)", 2, nsm, out, cyc);
  return 0;
}
