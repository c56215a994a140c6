// Cycles per tcgen05.mma.cta_group::2 (CTA pair, M = 256: 128 rows per CTA) at N = 64 / 128 / 256,
// SS and TS (A from TMEM): is the ~64-cycle per-instruction floor per SM or per pair instruction?
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_12131_b200/csrc/ptx.cuh"
using namespace btp;

__device__ __forceinline__ void umma_pair_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a_tmem), "l"(b_desc),
               "r"(idesc), "r"(acc));
}

template <int KIND, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* cyc, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t id_ss = make_idesc_bf16_f32(256, N, false, false);
    const uint32_t id_ts = make_idesc_bf16_f32(256, N, false, true);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const uint32_t off = (i & 3) * 32;
      if (KIND == 0) umma_bf16_pair(tmem + 256, make_sw128_desc(a + off, 16, 1024), make_sw128_desc(b + off, 16, 1024), id_ss, 1);
      if (KIND == 1) umma_pair_ts(tmem + 256, tmem + (i & 7) * 8, make_sw128_desc(b + (i & 7) * 2048, 16384, 1024), id_ts, 1);
    }
    umma_commit_pair_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x / 2] = t1 - t0;
  } else if (rank == 1 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_pair<512>(tmem); }
}

template <int KIND, int N>
void run(const char* name, int nsm, long long* cyc) {
  cudaFuncSetAttribute(k<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int n = 4096;
  k<KIND, N><<<nsm, 128, 70000>>>(cyc, n);
  k<KIND, N><<<nsm, 128, 70000>>>(cyc, n);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, cyc, nsm / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm / 2; ++i) mx = h[i] > mx ? h[i] : mx;
  const double fl = 2.0 * 256 * N * 16;
  printf("%-40s %6.1f clk / MMA  (%5.0f flop/clk/SM)  %s\n", name, (double)mx / n, fl * n / mx / 2,
         cudaGetErrorString(e));
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, 512 * 8);
  run<0, 64>("pair SS M256 N64", nsm, cyc);
  run<0, 128>("pair SS M256 N128", nsm, cyc);
  run<0, 256>("pair SS M256 N256", nsm, cyc);
  run<1, 64>("pair TS M256 N64 (A tmem)", nsm, cyc);
  run<1, 128>("pair TS M256 N128 (A tmem)", nsm, cyc);
  return 0;
}
