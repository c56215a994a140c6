// Cycles per tcgen05.mma of the shapes / operand sources the attention kernels issue (one CTA per SM,
// one thread issuing N back-to-back MMAs into one accumulator, commit + wait; clock64 around).
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_12131_b200/csrc/ptx.cuh"
using namespace btp;

template <int KIND>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t id_ss128 = make_idesc_bf16_f32(128, 128, false, false);
    const uint32_t id_ss256 = make_idesc_bf16_f32(128, 256, false, false);
    const uint32_t id_mn64 = make_idesc_bf16_f32(128, 64, true, true);
    const uint32_t id_ts64 = make_idesc_bf16_f32(128, 64, false, true);
    const uint32_t id_ts128 = make_idesc_bf16_f32(128, 128, false, true);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const uint32_t off = (i & 3) * 32;
      if (KIND == 0) umma_bf16(tmem, make_sw128_desc(a + off, 16, 1024), make_sw128_desc(b + off, 16, 1024), id_ss128, 1);
      if (KIND == 1) umma_bf16(tmem, make_sw128_desc(a + off, 16, 1024), make_sw128_desc(b + off, 16, 1024), id_ss256, 1);
      if (KIND == 2) umma_bf16(tmem + 256, make_sw128_desc(a + (i & 7) * 2048, 16384, 1024),
                               make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_mn64, 1);
      if (KIND == 3) umma_bf16_ts(tmem + 256, tmem + (i & 7) * 8, make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_ts64, 1);
      if (KIND == 5) umma_bf16_ts(tmem + 256 + (i & 1) * 64, tmem + (i & 7) * 8, make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_ts64, 1);
      if (KIND == 6) umma_bf16(tmem + 256 + (i & 1) * 64, make_sw128_desc(a + (i & 7) * 2048, 16384, 1024),
                               make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_mn64, 1);
      if (KIND == 7) umma_bf16(tmem + (i & 1) * 128, make_sw128_desc(a + off, 16, 1024), make_sw128_desc(b + off, 16, 1024), id_ss128, 1);
      if (KIND == 8) umma_bf16_ts(tmem + 256 + (i & 3) * 64, tmem + (i & 7) * 8, make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_ts64, 1);
      if (KIND == 4) umma_bf16_ts(tmem + 256, tmem + (i & 7) * 8, make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_ts128, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x < 512) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int KIND>
void run(const char* name, int nsm, long long* cyc, double flops_per) {
  cudaFuncSetAttribute(k<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int n = 4096;
  k<KIND><<<nsm, 128, 70000>>>(cyc, n);
  k<KIND><<<nsm, 128, 70000>>>(cyc, n);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-40s %6.1f clk / MMA  (%5.0f flop/clk/SM)  %s\n", name, (double)mx / n, flops_per * n / mx,
         cudaGetErrorString(e));
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, 512 * 8);
  run<0>("SS M128 N128 K16 (K-major both)", nsm, cyc, 2.0 * 128 * 128 * 16);
  run<1>("SS M128 N256 K16 (K-major both)", nsm, cyc, 2.0 * 128 * 256 * 16);
  run<2>("SS M128 N64 K16 (MN-major both)", nsm, cyc, 2.0 * 128 * 64 * 16);
  run<3>("TS M128 N64 K16 (A tmem, B MN-major)", nsm, cyc, 2.0 * 128 * 64 * 16);
  run<4>("TS M128 N128 K16 (A tmem, B MN-major)", nsm, cyc, 2.0 * 128 * 128 * 16);
  run<5>("TS M128 N64, 2 alternating accumulators", nsm, cyc, 2.0 * 128 * 64 * 16);
  run<8>("TS M128 N64, 4 alternating accumulators", nsm, cyc, 2.0 * 128 * 64 * 16);
  run<6>("SS N64 MN-major, 2 alternating accumulators", nsm, cyc, 2.0 * 128 * 64 * 16);
  run<7>("SS N128, 2 alternating accumulators", nsm, cyc, 2.0 * 128 * 128 * 16);
  return 0;
}
