// Per-SM issue rates of the instructions the attention softmax is built from (one 1024-thread block
// per SM, 8 independent chains per thread; clock64 around the loop). Prints ops / clk / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

#define N_IT 2048
template <int OP>
__global__ void __launch_bounds__(1024, 1) k(float* out, long long* cyc, float seed) {
  float v[8];
  uint32_t u[8];
  uint64_t d2[8];
  for (int i = 0; i < 8; ++i) { v[i] = seed * (threadIdx.x + i); u[i] = __float_as_uint(v[i]); d2[i] = u[i] * 0x100000001ull; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) & 7])); u[i] ^= r; }
      if (OP == 2) { uint32_t a = u[i] + 0x8000u, b = u[(i + 1) & 7] + 0x8000u; uint32_t r;
                     asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b)); u[i] = r; }
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
      if (OP == 4) { uint64_t d; asm volatile("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(v[i]), "f"(v[(i + 1) & 7]));
                     asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d)); float a, b;
                     asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(d)); v[i] = a + b; }
      if (OP == 5) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(u[i]), "r"(u[(i + 1) & 7])); u[i] = r; }
      if (OP == 6) asm volatile("add.u32 %0, %0, 0x8000;" : "+r"(u[i]));
      if (OP == 7) asm volatile("mad.lo.u32 %0, %0, 3, 0x8000;" : "+r"(u[i]));
      if (OP == 9) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d2[i]) : "l"(d2[(i + 1) & 7]), "l"(d2[(i + 2) & 7]));
      if (OP == 10) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(d2[i]) : "l"(d2[(i + 3) & 7]));
      if (OP == 11) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 1) & 7]), "f"(v[(i + 2) & 7]));
      if (OP == 12) { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 1) & 7]), "f"(v[(i + 2) & 7])); }
      if (OP == 13) { float e; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(v[i]));
                      asm volatile("fma.rn.f32 %0, %1, %0, %0;" : "+f"(v[i]) : "f"(e));
                      uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e), "f"(v[i])); u[i] += r; }
      if (OP == 8) { uint32_t r; asm volatile("cvt.rn.satfinite.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) & 7])); u[i] ^= r; }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i] + __uint_as_float(u[i]) + __uint_as_float((uint32_t)d2[i]);
  out[blockIdx.x * 1024 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int nsm, float* out, long long* cyc) {
  k<OP><<<nsm, 1024>>>(out, cyc, 1e-3f);
  k<OP><<<nsm, 1024>>>(out, cyc, 1e-3f);
  cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = 1024.0 * N_IT * 8;
  printf("%-34s %7.1f thread-instr / clk / SM\n", name, ops / mx);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, nsm * 1024 * 4);
  cudaMalloc(&cyc, nsm * 8);
  run<0>("ex2.approx.ftz.f32 (MUFU)", nsm, out, cyc);
  run<1>("cvt.rn.bf16x2.f32 (+LOP)", nsm, out, cyc);
  run<8>("cvt.rn.satfinite.bf16x2.f32 (+LOP)", nsm, out, cyc);
  run<2>("2x iadd + prmt (manual pack)", nsm, out, cyc);
  run<3>("fma.rn.f32", nsm, out, cyc);
  run<4>("fma.rn.f32x2 (+mov, fadd)", nsm, out, cyc);
  run<5>("prmt.b32", nsm, out, cyc);
  run<6>("add.u32", nsm, out, cyc);
  run<7>("mad.lo.u32", nsm, out, cyc);
  run<9>("fma.rn.f32x2 (independent)", nsm, out, cyc);
  run<10>("mul.rn.f32x2 (independent)", nsm, out, cyc);
  run<11>("max.f32 3-input", nsm, out, cyc);
  run<12>("fma.rn.f32 (3 distinct regs)", nsm, out, cyc);
  run<13>("ex2 + fma + cvt.bf16x2 (per group)", nsm, out, cyc);
  return 0;
}
