// The hd-64 attention backward's per-query-tile tcgen05 sequence in isolation (one CTA / SM, one
// thread issuing, operands resident): [1] 4x SS N128, [3] 8x TS N64, [2] 4x SS N128, [4] 8x SS N64
// (A K-major, B MN-major), [5] 8x SS N64 (both MN-major), with the kernel's commits. Variants reorder /
// drop pieces to see what the sequence costs versus the sum of its instructions.
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_12131_b200/csrc/ptx.cuh"
using namespace btp;

template <int KIND>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t sK = smem_u32(smem), sV = sK + 16384, sQ = sK + 32768, sdO = sK + 49152, sdS = sK + 65536;
    const uint32_t id_ss = make_idesc_bf16_f32(128, 128, false, false);
    const uint32_t id_ts = make_idesc_bf16_f32(128, 64, false, true);
    const uint32_t id_dq = make_idesc_bf16_f32(128, 64, true, true);
    const uint32_t tS = tm, tP = tm + 128, tdP = tm + 192, tdV = tm + 320, tdK = tm + 384, tdQ = tm + 448;
    auto m1 = [&]() { for (int k = 0; k < 4; ++k) umma_bf16(tS, make_sw128_desc(sK + k * 32, 16, 1024), make_sw128_desc(sQ + k * 32, 16, 1024), id_ss, k > 0); };
    auto m2 = [&]() { for (int k = 0; k < 4; ++k) umma_bf16(tdP, make_sw128_desc(sV + k * 32, 16, 1024), make_sw128_desc(sdO + k * 32, 16, 1024), id_ss, k > 0); };
    auto m3 = [&]() { for (int k = 0; k < 8; ++k) umma_bf16_ts(tdV, tP + (k >> 2) * 32 + (k & 3) * 8, make_sw128_desc(sdO + k * 2048, 16384, 1024), id_ts, 1); };
    auto m4 = [&]() { for (int k = 0; k < 8; ++k) umma_bf16(tdK, make_sw128_desc(sdS + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), make_sw128_desc(sQ + k * 2048, 16384, 1024), id_ts, 1); };
    auto m5 = [&]() { for (int k = 0; k < 8; ++k) umma_bf16(tdQ, make_sw128_desc(sdS + k * 2048, 16384, 1024), make_sw128_desc(sK + k * 2048, 16384, 1024), id_dq, k > 0); };
    long long t0 = clock64();
    for (int i = 0; i < tiles; ++i) {
      if (KIND == 0) { m1(); umma_commit(&bar[0]); m3(); umma_commit(&bar[1]); m2(); umma_commit(&bar[2]); m4(); umma_commit(&bar[3]); m5(); umma_commit(&bar[4]); umma_commit(&bar[5]); }
      if (KIND == 1) { m1(); m3(); m2(); m4(); m5(); }                          // no commits
      if (KIND == 2) { m1(); m2(); }                                          // the two N128 products
      if (KIND == 3) { m3(); m4(); m5(); }                                    // the three N64 products
      if (KIND == 4) { m3(); }
      if (KIND == 5) { m4(); }
      if (KIND == 6) { m5(); }
      if (KIND == 7) { m1(); }
    }
    umma_commit(&bar[7]);
    mbar_wait(&bar[7], 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

template <int KIND>
void run(const char* name, int nsm, long long* cyc, int mmas) {
  cudaFuncSetAttribute(k<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const int tiles = 512;
  k<KIND><<<nsm, 128, 200000>>>(cyc, tiles);
  k<KIND><<<nsm, 128, 200000>>>(cyc, tiles);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-44s %7.1f clk / tile  (%5.1f clk / MMA)  %s\n", name, (double)mx / tiles, (double)mx / tiles / mmas,
         cudaGetErrorString(e));
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, 512 * 8);
  run<0>("full tile sequence + commits", nsm, cyc, 32);
  run<1>("full tile sequence, no commits", nsm, cyc, 32);
  run<2>("[1]+[2] (SS N128 x 8)", nsm, cyc, 8);
  run<3>("[3]+[4]+[5] (N64 x 24)", nsm, cyc, 24);
  run<4>("[3] TS N64 x 8", nsm, cyc, 8);
  run<5>("[4] SS N64 A-Kmaj B-MNmaj x 8", nsm, cyc, 8);
  run<6>("[5] SS N64 both MN-major x 8", nsm, cyc, 8);
  run<7>("[1] SS N128 x 4", nsm, cyc, 4);
  return 0;
}
