// Persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
//   C[M,N] = epilogue( sum_k A[m,k] * B[n,k] )
//
// One launch serves up to kMaxProblems independent problems (the grouped / batched
// GEMMs of the BTP chunks: q|k|v or gate|up up-projections, reference
// simulator.py:655-668 `up_gemms`, tensor.py:97-112 `batched_matmul`) and optional
// split-K (weight gradients, whose reduction runs over the T tokens).
//
// Operands are staged by TMA into 128B-swizzled shared memory; either operand may be
// K-major (row-major [rows, K]) or MN-major (row-major [K, rows]); the UMMA descriptor
// "major" bits absorb the transpose so dgrad/wgrad never materialise a transposed copy.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4..w7 epilogue (TMEM lane quarter = warp % 4). The accumulator is double-buffered in
// TMEM (2 x BN columns) so the epilogue of tile i overlaps the mainloop of tile i+1.
//
// Epilogue: TMEM -> registers (scale / residual / convert) -> 128B-swizzled smem staging
// (32 rows x 128 B per warp, double-buffered) -> TMA bulk tensor store. Split-K partials use
// the TMA reduce-add form (fp32 add performed in L2) into a zero-initialised fp32 output, so
// there are no partial slabs and no separate reduction pass.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "btp_internal.h"
#include "ptx.cuh"

namespace btp {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kMaxProblems = 8;  // DevParams (~8 KB with 8) travels as a >4 KB kernel parameter (CUDA >= 12.1)
constexpr int kThreads = 256;
constexpr int kEpiStageBytes = 32 * 128;              // one warp's 32 rows x 128 B chunk

// Epilogue modes (per problem)
constexpr int kEpiStore = 0;      // C = scale * acc (+ resid if given); store or reduce-add
constexpr int kEpiSigma = 1;      // rank-r boundary at TP=1: C = z = scale*acc, C2 = crossgate(z)
constexpr int kEpiSwigluBwd = 2;  // acc = dact; aux g (resid slot), u (aux2): C = dg, C2 = du

struct alignas(64) DevProblem {
  CUtensorMap tma_a;
  CUtensorMap tma_b;
  CUtensorMap tma_c;
  CUtensorMap tma_r;   // residual / first aux input (bf16, same box as the bf16 output)
  CUtensorMap tma_c2;  // second output (swiglu-bwd: du)
  CUtensorMap tma_r2;  // second aux input (swiglu-bwd: u)
  int epi;
  const float* row_scale;
  const float* col_scale;
  const __nv_bfloat16* resid;
  long long ld_resid;
  int M, N, K;
  int m_tiles, n_tiles, splits, kb_per_split, k_blocks;
  int tile_start;
  int out_fp32;
  int reduce_add;   // split-K: TMA reduce-add into the fp32 output
  int a_mn, b_mn;   // operand majors (per problem: a launch may mix dgrad and wgrad problems)
  uint32_t idesc;   // tcgen05 instruction descriptor for this problem
  float alpha;
  int sig_half;     // kEpiSigma: r/2; an N tile = BN/2 "u" columns + the BN/2 "v" columns r/2 later
  int scatter_col0; // scatter mode: this problem's first column in the owners' buffers
  char* c_ptr;      // st.global epilogue stores: outputs and row strides (elements)
  char* c2_ptr;
  long long ldc, ldc2;
};

constexpr int kMaxOwners = 8;

struct DevParams {
  DevProblem prob[kMaxProblems];
  int num_problems;
  int total_tiles;
  // Scatter mode (the GEMM half of a BTP chunk boundary over peer memory): every 32-row x 32-column
  // fp32 output chunk is TMA reduce-added (cp.reduce.async.bulk.tensor .add, the fp32 add performed
  // at the destination) into the buffer of the rank owning those rows — rows [o * scatter_rows,
  // (o + 1) * scatter_rows) belong to rank o — instead of being stored locally: the reduce-scatter
  // of the row-parallel partial happens tile by tile inside the GEMM, over NVLink. fp32 because
  // sm_100a's tensor reduce has no bf16 add, and it keeps the cross-rank sum at one rounding
  // (per-row register red.add was 3.6x slower: one row per lane is uncoalesced).
  int scatter_n;
  int scatter_rows;
  // 1: plain stores leave the epilogue as coalesced st.global (4 rows x 128 B per warp instruction)
  // from the swizzled staging chunk instead of TMA bulk-tensor stores — the TMA unit then only moves
  // operands (and the residual), which is what bounds the K = 512 GEMMs (TMA bytes per tile).
  int st_global;
  CUtensorMap scatter[kMaxOwners];
};

// kSlots: staging slots per chunk buffer (2 for the two-input / two-output swiglu-bwd epilogue,
// which trades mainloop stages for epilogue staging). kSlots == 4 is the residual layout: four
// single-slot chunk buffers per warp, so a tile's whole residual (<= 4 x 64 columns) is TMA-loaded
// in one go and each chunk is added and stored in place.
// kSlots == 5 is the pipelined residual layout (kResPipe, CTA pairs): per epilogue warp four
// residual chunk slots owned by a dedicated residual-producer warp (warp 3) plus two output
// staging buffers. The producer refills a slot with the NEXT tile's residual chunk as soon as the
// epilogue has read it into registers, so a tile's residual is in flight for a whole tile period
// instead of being issued when the tile's epilogue starts (the kSlots == 4 layout's exposed latency).
// kPair: CTA-pair mode (cluster of 2, tcgen05.mma.cta_group::2): a 256 x BN tile per pair,
// each CTA holding 128 rows of A and BN/2 rows of B per stage and its own 128 x BN accumulator.
// Halving the per-CTA B tile buys a deeper smem pipeline (up to 8 stages).
template <int BN, int kSlots, bool kPair>
struct Cfg {
  static constexpr int kBRows = kPair ? BN / 2 : BN;
  static constexpr int kTileM = kPair ? 2 * kBM : kBM;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = (2 * BN <= 256) ? 256 : 512;  // double-buffered accumulator (pow2 alloc)
  static constexpr bool kResPipe = kSlots == 5;
  static constexpr int kEpiWarpBytes =
      (kResPipe ? 6 : (kSlots == 4 ? 4 : 2 * kSlots)) * kEpiStageBytes;  // chunk buffers
  static constexpr int kEpiBytes = 4 * kEpiWarpBytes;
  static constexpr int kBarrierBytes = kResPipe ? 1024 : 512;
  static constexpr int kAvail = 232448 - 1024 - kEpiBytes - kBarrierBytes;
  static constexpr int kStages = (kAvail / kStageBytes) > 8 ? 8 : (kAvail / kStageBytes);
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kEpiBytes + kBarrierBytes;
};

struct TileCoord {
  int p, split, m_blk, n_blk;
};

__device__ __forceinline__ TileCoord decode_tile(const DevParams& P, int tile) {
  int p = 0;
#pragma unroll
  for (int i = 1; i < kMaxProblems; ++i)
    if (i < P.num_problems && tile >= P.prob[i].tile_start) p = i;
  const DevProblem& pr = P.prob[p];
  int local = tile - pr.tile_start;
  const int per_split = pr.m_tiles * pr.n_tiles;
  TileCoord t;
  t.p = p;
  t.split = local / per_split;
  local -= t.split * per_split;
  t.m_blk = local / pr.n_tiles;
  t.n_blk = local - t.m_blk * pr.n_tiles;
  return t;
}

template <int BN, int kSlots, bool kPair>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ DevParams P) {
  using C = Cfg<BN, kSlots, kPair>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* sEpi = smem + C::kStages * C::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sEpi + C::kEpiBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar_all = tempty_bar + 2;  // 4 epilogue warps x (2, or 4 when kSlots == 4) buffers
  // kResPipe: residual slot (warp q, chunk c) -> full / empty barriers at index q * 4 + c
  uint64_t* res_full = aux_bar_all + 16;
  uint64_t* res_empty = res_full + (C::kResPipe ? 16 : 0);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_empty + (C::kResPipe ? 16 : 0));

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  // pair mode: rank within the CTA pair; tiles are distributed over pairs
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const int unit = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int n_units = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < P.num_problems; ++i) {
      tma_prefetch_desc(&P.prob[i].tma_a);
      tma_prefetch_desc(&P.prob[i].tma_b);
      tma_prefetch_desc(&P.prob[i].tma_c);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      // one arrival per epilogue warp (pair: both CTAs' four warps release the leader's buffer)
      mbar_init(&tempty_bar[b], kPair ? 8 : 4);
    }
    for (int b = 0; b < 16; ++b) mbar_init(&aux_bar_all[b], 1);
    if constexpr (C::kResPipe) {
      for (int b = 0; b < 16; ++b) {
        mbar_init(&res_full[b], 1);
        mbar_init(&res_empty[b], 1);  // the owning epilogue warp's lane 0
      }
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (kPair) tmem_alloc_pair<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // peer barriers must exist before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = unit; tile < P.total_tiles; tile += n_units) {
        const TileCoord tc = decode_tile(P, tile);
        const DevProblem& pr = P.prob[tc.p];
        const int m0 = tc.m_blk * C::kTileM + (int)rank * kBM;     // this CTA's 128 rows of A
        const int n0 = tc.n_blk * BN + (int)rank * (BN - C::kBRows);  // this CTA's share of B
        const int kb0 = tc.split * pr.kb_per_split;
        const int kb1 = min(kb0 + pr.kb_per_split, pr.k_blocks);
        // sigma tiles pair column blocks [u0, u0 + BN/2) and [u0 + r/2, ...) of B (K-major)
        int u0 = 0;
        if (pr.epi == kEpiSigma) {
          const int npp = 2 * pr.sig_half / BN;
          const int proj = tc.n_blk / npp;
          u0 = proj * 2 * pr.sig_half + (tc.n_blk - proj * npp) * (BN / 2);
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          // pair: both CTAs' bytes complete on the leader's barrier, which expects both halves
          const uint32_t fbar = kPair ? (smem_u32(&full_bar[stage]) & kPeerBitMask) : smem_u32(&full_bar[stage]);
          if (!kPair || rank == 0) mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes * (kPair ? 2 : 1));
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
          const int k0 = kb * kBK;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if constexpr (kPair) tma_load_2d_pair(dst, m, fbar, c0, c1);
            else tma_load_2d(dst, m, &full_bar[stage], c0, c1);
          };
          if (!pr.a_mn) {
            load(a_dst, &pr.tma_a, k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < kBM / 64; ++c) load(a_dst + c * 64 * kBK * 2, &pr.tma_a, m0 + c * 64, k0);
          }
          if (pr.epi == kEpiSigma) {
            if constexpr (kPair) {
              load(b_dst, &pr.tma_b, k0, u0 + (int)rank * pr.sig_half);  // leader: u rows, peer: v rows
            } else {
              load(b_dst, &pr.tma_b, k0, u0);
              load(b_dst + (BN / 2) * kBK * 2, &pr.tma_b, k0, u0 + pr.sig_half);
            }
          } else if (!pr.b_mn) {
            load(b_dst, &pr.tma_b, k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < C::kBRows / 64; ++c) load(b_dst + c * 64 * kBK * 2, &pr.tma_b, n0 + c * 64, k0);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && (!kPair || rank == 0)) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = unit; tile < P.total_tiles; tile += n_units, ++it) {
      const TileCoord tc = decode_tile(P, tile);
      const DevProblem& pr = P.prob[tc.p];
      const int kb0 = tc.split * pr.kb_per_split;
      const int kb1 = min(kb0 + pr.kb_per_split, pr.k_blocks);
      const int buf = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
          // K-major: advance 32 B along the swizzled row; MN-major: advance 16 rows (2 KB)
          const uint32_t a_step = pr.a_mn ? 16 * 128 : 32, b_step = pr.b_mn ? 16 * 128 : 32;
          const uint32_t a_lbo = pr.a_mn ? 64 * kBK * 2 : 16, b_lbo = pr.b_mn ? 64 * kBK * 2 : 16;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t a_desc = make_sw128_desc(a_base + k * a_step, a_lbo, 1024);
            const uint64_t b_desc = make_sw128_desc(b_base + k * b_step, b_lbo, 1024);
            if constexpr (kPair) umma_bf16_pair(d_tmem, a_desc, b_desc, pr.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else umma_bf16(d_tmem, a_desc, b_desc, pr.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (kPair) umma_commit_pair_mc(&empty_bar[stage], 0x3);  // frees the slot in both CTAs
          else umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) {
        if constexpr (kPair) umma_commit_pair_mc(&tfull_bar[buf], 0x3);
        else umma_commit(&tfull_bar[buf]);
      }
      __syncwarp();
    }
  } else if (C::kResPipe && warp == 3) {
    // ------------------------------------------------------------ residual producer (kResPipe)
    // Walks the same tile sequence as the epilogue; slot (q, c) of the next residual tile is
    // refilled as soon as epilogue warp q has read chunk c of the previous one.
    if (elect_one()) {
      uint32_t ph = 0u;  // bit s: parity flips per use of slot s
      for (int tile = unit; tile < P.total_tiles; tile += n_units) {
        const TileCoord tc = decode_tile(P, tile);
        const DevProblem& pr = P.prob[tc.p];
        if (pr.resid == nullptr) continue;
        const int m0 = tc.m_blk * C::kTileM + (int)rank * kBM, n0 = tc.n_blk * BN;
        const int n_valid = min(BN, pr.N - n0);
        for (int c = 0; c < 4 && c * 64 < n_valid; ++c) {
#pragma unroll 1
          for (int qq = 0; qq < 4; ++qq) {
            const int sl = qq * 4 + c;
            mbar_wait(&res_empty[sl], ((ph >> sl) & 1u) ^ 1u);
            ph ^= 1u << sl;
            mbar_arrive_expect_tx(&res_full[sl], kEpiStageBytes);
            tma_load_2d(sEpi + qq * C::kEpiWarpBytes + c * kEpiStageBytes, &pr.tma_r, &res_full[sl], n0 + c * 64,
                        m0 + qq * 32);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter == rows [32q, 32q+32) of the tile
    uint8_t* stage_ptr0 = sEpi + q * C::kEpiWarpBytes;
    const uint32_t stage0 = smem_u32(stage_ptr0);
    const uint32_t row_sw = lane & 7;  // 128B swizzle: 16B chunk j of row i lives at chunk j ^ (i % 8)
    uint64_t* aux_bar = aux_bar_all + q * (kSlots == 4 ? 4 : 2);  // one per staging buffer of this warp
    uint32_t res_phase = 0u;  // kSlots == 4: bit c = parity of the next wait on aux_bar[c]
    uint32_t aux_phase = 0u;  // bit b: parity of the next wait on aux_bar[b]
    // staging slot s of buffer b (each slot = one 32-row x 128 B chunk)
    auto slot_ptr = [&](int b, int s) { return stage_ptr0 + (b * kSlots + s) * kEpiStageBytes; };
    // coalesced store of one staged 32-row x 128 B chunk (128B-swizzled) at (row0, col0) of an
    // output with row stride ld elements of esz bytes; rows >= M and columns >= N are skipped (N % 8
    // == 0, so a 16-byte segment never straddles N). The warp reads the staging synchronously, so
    // the buffer is free again after the following __syncwarp.
    auto store_chunk = [&](const uint8_t* sbuf, char* base, long long ld, int esz, int M, int N, int row0, int col0) {
      const uint32_t sa = smem_u32(sbuf);
      const int seg = (int)(lane & 7);
      const int cpos = col0 + seg * (16 / esz);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = j * 4 + (int)(lane >> 3);
        const uint4 v = ld_shared_v4(sa + i * 128 + ((seg ^ (i & 7)) << 4));
        const int row = row0 + i;
        if (row < M && cpos < N) st_global_v4(base + ((long long)row * ld + cpos) * esz, v);
      }
      __syncwarp();
    };
    // lane 0: TMA-load the aux chunk(s) for output column `col` into buffer b
    auto issue_aux = [&](const DevProblem& pr, int b, int col, int row0) {
      const int naux = pr.epi == kEpiSwigluBwd ? 2 : 1;
      bulk_wait_read<0>();  // every earlier store has finished reading its staging slots
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&aux_bar[b], naux * kEpiStageBytes);
      tma_load_2d(slot_ptr(b, 0), &pr.tma_r, &aux_bar[b], col, row0);
      if (naux == 2) tma_load_2d(slot_ptr(b, 1), &pr.tma_r2, &aux_bar[b], col, row0);
    };
    // hand TMEM accumulator buffer `b` back to the MMA warp: every lane's tcgen05.ld has completed
    // (tcgen05.wait::ld), the warp converges, and ONE lane orders and arrives for the warp
    auto release_tmem = [&](int b) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair) mbar_arrive_cluster(&tempty_bar[b], 0);
        else mbar_arrive(&tempty_bar[b]);
      }
    };
    int it = 0;
    int chunk_seq = 0;  // running chunk counter -> staging buffer parity
    for (int tile = unit; tile < P.total_tiles; tile += n_units, ++it) {
      const TileCoord tc = decode_tile(P, tile);
      const DevProblem& pr = P.prob[tc.p];
      const int buf = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = tc.m_blk * C::kTileM + (int)rank * kBM, n0 = tc.n_blk * BN;  // this CTA's 128 rows
      const int n_valid = min(BN, pr.N - n0);
      const int cols_per_chunk = pr.out_fp32 ? 32 : 64;  // 128 bytes of output per row
      const int out_row0 = m0 + q * 32;
      // aux tiles (residual, or g/u for swiglu-bwd) ride the staging buffers (bf16 out only)
      const bool aux = pr.resid != nullptr;
      const bool swb = pr.epi == kEpiSwigluBwd;
      if constexpr (C::kResPipe) {
        // residual chunks arrive through the producer warp's slots
      } else if constexpr (kSlots == 4) {
        // the tile's whole residual in flight at once (one latency per tile, not per chunk), as
        // soon as the previous tile's stores have read the buffers
        if (lane == 0) {
          bulk_wait_read<0>();
          if (aux) {
            fence_proxy_async_smem();
            for (int c = 0; c < 4 && c * 64 < n_valid; ++c) {
              mbar_arrive_expect_tx(&aux_bar[c], kEpiStageBytes);
              tma_load_2d(stage_ptr0 + c * kEpiStageBytes, &pr.tma_r, &aux_bar[c], n0 + c * 64, out_row0);
            }
          }
        }
        __syncwarp();
      } else if (aux && lane == 0) {
        issue_aux(pr, chunk_seq & 1, n0, out_row0);  // prefetch under the mainloop
      }
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < pr.M;
      float rscale = pr.alpha;
      if (pr.row_scale != nullptr && row_ok) rscale *= pr.row_scale[row];
      if constexpr (C::kResPipe) {
        // bf16 output, 64-column chunks c = 0..3: TMEM -> registers (+ residual slot c, released to
        // the producer right after the read) -> output staging buffer (double-buffered) -> TMA store
#pragma unroll 1
        for (int c = 0; c * 64 < n_valid; ++c, ++chunk_seq) {
          const int c0 = c * 64;
          float v[64];
          {
            uint32_t r[64];
            tmem_ld_32x32b_x64(tmem_base + ((q * 32u) << 16) + buf * BN + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]) * rscale;
          }
          if (c0 + 64 >= n_valid) release_tmem(buf);
          const int col = n0 + c0;
          if (pr.col_scale != nullptr) {
            const int lim = min(64, n_valid - c0);
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < lim) v[j] *= __ldg(pr.col_scale + col + j);
          }
          if (aux) {
            const int sl = (int)q * 4 + c;
            mbar_wait(&res_full[sl], (res_phase >> c) & 1u);
            res_phase ^= 1u << c;
            const uint32_t raddr = smem_u32(stage_ptr0 + c * kEpiStageBytes) + lane * 128;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const uint4 rv = ld_shared_v4(raddr + ((g ^ row_sw) << 4));
              const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                v[g * 8 + 2 * h] += bf16_lo(w[h]);
                v[g * 8 + 2 * h + 1] += bf16_hi(w[h]);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&res_empty[sl]);  // every lane has its residual in registers
          }
          uint8_t* ob = stage_ptr0 + (4 + (chunk_seq & 1)) * kEpiStageBytes;
          const uint32_t row_addr = smem_u32(ob) + lane * 128;
          if (lane == 0) bulk_wait_read<1>();  // the store issued two chunks ago has read this buffer
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(row_addr + ((j ^ row_sw) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                         pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                         pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          if (P.st_global) {
            __syncwarp();
            store_chunk(ob, pr.c_ptr, pr.ldc, 2, pr.M, pr.N, out_row0, col);
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&pr.tma_c, ob, col, out_row0);
            bulk_commit();
          }
        }
        continue;
      } else if constexpr (kSlots == 4) {
        // bf16 output, 64-column chunks c = 0..3: residual (if any) landed in buffer c; the sum is
        // written back in place and TMA-stored from there
#pragma unroll 1
        for (int c = 0; c * 64 < n_valid; ++c) {
          const int c0 = c * 64;
          uint8_t* cb = stage_ptr0 + c * kEpiStageBytes;
          const uint32_t row_addr = smem_u32(cb) + lane * 128;
          if (aux) {
            mbar_wait(&aux_bar[c], (res_phase >> c) & 1u);
            res_phase ^= 1u << c;
          }
          float v[64];
          {
            uint32_t r[64];
            tmem_ld_32x32b_x64(tmem_base + ((q * 32u) << 16) + buf * BN + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]) * rscale;
          }
          if (c0 + 64 >= n_valid) release_tmem(buf);
          const int col = n0 + c0;
          if (pr.col_scale != nullptr) {
            const int lim = min(64, n_valid - c0);
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < lim) v[j] *= __ldg(pr.col_scale + col + j);
          }
          if (aux) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const uint4 rv = ld_shared_v4(row_addr + ((g ^ row_sw) << 4));
              const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                v[g * 8 + 2 * h] += bf16_lo(w[h]);
                v[g * 8 + 2 * h + 1] += bf16_hi(w[h]);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(row_addr + ((j ^ row_sw) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                         pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                         pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          if (P.st_global) {
            __syncwarp();
            store_chunk(cb, pr.c_ptr, pr.ldc, 2, pr.M, pr.N, out_row0, col);
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&pr.tma_c, cb, col, out_row0);
            bulk_commit();
          }
        }
        continue;
      }
      if (kSlots == 2 && pr.epi == kEpiSigma) {  // (launched with two staging slots per buffer)
        // accumulator columns [0, BN/2) = u block, [BN/2, BN) = v block of the same projection.
        // Per 64-column step: z_u, z_v -> C from staging buffer 0 (two slots), then
        // a_u = silu(u) v, a_v = silu(v) u -> C2 from buffer 1; each buffer is reused only after
        // its previous TMA store group has read it (one group stays in flight).
        const int hb = BN / 2;
        const int npp = 2 * pr.sig_half / BN;
        const int proj = tc.n_blk / npp;
        const int u0 = proj * 2 * pr.sig_half + (tc.n_blk - proj * npp) * hb;
        const int v0 = u0 + pr.sig_half;
        uint8_t* sz0 = slot_ptr(0, 0);
        uint8_t* sz1 = slot_ptr(0, kSlots - 1);
        uint8_t* sa0 = slot_ptr(1, 0);
        uint8_t* sa1 = slot_ptr(1, kSlots - 1);
        const uint32_t rz0 = smem_u32(sz0) + lane * 128, rz1 = smem_u32(sz1) + lane * 128;
        const uint32_t ra0 = smem_u32(sa0) + lane * 128, ra1 = smem_u32(sa1) + lane * 128;
        const uint32_t tbase = tmem_base + ((q * 32u) << 16) + buf * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < hb; c0 += 64) {
          uint32_t zu[32], zv[32];
          {
            uint32_t r[64];
            tmem_ld_32x32b_x64(tbase + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              zu[j] = pack_bf16(__uint_as_float(r[2 * j]) * rscale, __uint_as_float(r[2 * j + 1]) * rscale);
            tmem_ld_32x32b_x64(tbase + hb + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              zv[j] = pack_bf16(__uint_as_float(r[2 * j]) * rscale, __uint_as_float(r[2 * j + 1]) * rscale);
          }
          if (c0 + 64 >= hb) release_tmem(buf);  // accumulator fully in registers: free the TMEM buffer now
          if (lane == 0) bulk_wait_read<1>();  // the z buffer's previous group has been read
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            st_shared_v4(rz0 + ((g ^ row_sw) << 4), zu[4 * g], zu[4 * g + 1], zu[4 * g + 2], zu[4 * g + 3]);
            st_shared_v4(rz1 + ((g ^ row_sw) << 4), zv[4 * g], zv[4 * g + 1], zv[4 * g + 2], zv[4 * g + 3]);
          }
          if (P.st_global) {
            __syncwarp();
            store_chunk(sz0, pr.c_ptr, pr.ldc, 2, pr.M, pr.N, out_row0, u0 + c0);
            store_chunk(sz1, pr.c_ptr, pr.ldc, 2, pr.M, pr.N, out_row0, v0 + c0);
          } else {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&pr.tma_c, sz0, u0 + c0, out_row0);
              tma_store_2d(&pr.tma_c, sz1, v0 + c0, out_row0);
              bulk_commit();
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float ul = bf16_lo(zu[j]), uh = bf16_hi(zu[j]);
            const float vl = bf16_lo(zv[j]), vh = bf16_hi(zv[j]);
            zu[j] = pack_bf16(silu_crossgate<__nv_bfloat16>(ul) * vl, silu_crossgate<__nv_bfloat16>(uh) * vh);
            zv[j] = pack_bf16(silu_crossgate<__nv_bfloat16>(vl) * ul, silu_crossgate<__nv_bfloat16>(vh) * uh);
          }
          if (lane == 0) bulk_wait_read<1>();  // the a buffer's previous group has been read
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            st_shared_v4(ra0 + ((g ^ row_sw) << 4), zu[4 * g], zu[4 * g + 1], zu[4 * g + 2], zu[4 * g + 3]);
            st_shared_v4(ra1 + ((g ^ row_sw) << 4), zv[4 * g], zv[4 * g + 1], zv[4 * g + 2], zv[4 * g + 3]);
          }
          if (P.st_global) {
            __syncwarp();
            store_chunk(sa0, pr.c2_ptr, pr.ldc2, 2, pr.M, pr.N, out_row0, u0 + c0);
            store_chunk(sa1, pr.c2_ptr, pr.ldc2, 2, pr.M, pr.N, out_row0, v0 + c0);
          } else {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&pr.tma_c2, sa0, u0 + c0, out_row0);
              tma_store_2d(&pr.tma_c2, sa1, v0 + c0, out_row0);
              bulk_commit();
            }
          }
        }
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < n_valid; c0 += cols_per_chunk, ++chunk_seq) {
        const int b = chunk_seq & 1;
        const uint32_t stage = smem_u32(slot_ptr(b, 0));
        if (!aux) {
          // the TMA store issued two chunks ago used this staging buffer: it must have read it
          if (lane == 0) bulk_wait_read<kSlots>();
        } else {
          // prefetch the next chunk's aux into the other buffer, then wait for this one
          if (lane == 0 && c0 + cols_per_chunk < n_valid) issue_aux(pr, b ^ 1, n0 + c0 + cols_per_chunk, out_row0);
          mbar_wait(&aux_bar[b], (aux_phase >> b) & 1u);
          aux_phase ^= 1u << b;
        }
        __syncwarp();
        float v[64];
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * BN + c0;
        if (!pr.out_fp32) {
          uint32_t r[64];
          tmem_ld_32x32b_x64(taddr, r);  // one TMEM round trip per 64-column chunk
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]) * rscale;
        } else {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * rscale;
        }
        // last chunk of the tile in registers: the MMA warp may overwrite this TMEM buffer while
        // the chunk is still being converted and stored
        if (c0 + cols_per_chunk >= n_valid) release_tmem(buf);
        const int col = n0 + c0;
        if (pr.col_scale != nullptr) {
          const int lim = min(cols_per_chunk, n_valid - c0);
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < lim) v[j] *= __ldg(pr.col_scale + col + j);
        }
        const uint32_t row_addr = stage + lane * 128;
        if (swb) {
          // acc = dact; slot 0 holds g, slot 1 holds u: dg = dact*u*silu'(g) -> slot 0, du = dact*silu(g) -> slot 1
          const uint32_t row_addr2 = smem_u32(slot_ptr(b, 1)) + lane * 128;
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            const uint32_t off = ((g8 ^ row_sw) << 4);
            const uint4 gv = ld_shared_v4(row_addr + off);
            const uint4 uv = ld_shared_v4(row_addr2 + off);
            const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
            const uint32_t uw[4] = {uv.x, uv.y, uv.z, uv.w};
            uint32_t dgw[4], duw[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              float dg2[2], du2[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const float gg = e ? bf16_hi(gw[h]) : bf16_lo(gw[h]);
                const float uu = e ? bf16_hi(uw[h]) : bf16_lo(uw[h]);
                const float da = v[g8 * 8 + 2 * h + e];
                const float sg = sigmoidf_safe(gg);
                dg2[e] = da * uu * sg * (1.0f + gg * (1.0f - sg));
                du2[e] = da * gg * sg;
              }
              dgw[h] = pack_bf16(dg2[0], dg2[1]);
              duw[h] = pack_bf16(du2[0], du2[1]);
            }
            st_shared_v4(row_addr + off, dgw[0], dgw[1], dgw[2], dgw[3]);
            st_shared_v4(row_addr2 + off, duw[0], duw[1], duw[2], duw[3]);
          }
          if (P.st_global) {
            __syncwarp();
            store_chunk(slot_ptr(b, 0), pr.c_ptr, pr.ldc, 2, pr.M, pr.N, out_row0, col);
            store_chunk(slot_ptr(b, 1), pr.c2_ptr, pr.ldc2, 2, pr.M, pr.N, out_row0, col);
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&pr.tma_c, slot_ptr(b, 0), col, out_row0);
            tma_store_2d(&pr.tma_c2, slot_ptr(b, 1), col, out_row0);
            bulk_commit();
          }
          continue;
        }
        if (aux) {
          // residual chunk (same swizzled layout as the output), read then overwritten in place
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const uint4 rv = ld_shared_v4(row_addr + ((g ^ row_sw) << 4));
            const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              v[g * 8 + 2 * h] += bf16_lo(w[h]);
              v[g * 8 + 2 * h + 1] += bf16_hi(w[h]);
            }
          }
        }
        if (pr.out_fp32) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(row_addr + ((j ^ row_sw) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                         __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(row_addr + ((j ^ row_sw) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                         pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                         pack_bf16(v[8 * j + 6], v[8 * j + 7]));
        }
        if (P.st_global && P.scatter_n == 0 && !pr.reduce_add) {
          __syncwarp();
          store_chunk(slot_ptr(b, 0), pr.c_ptr, pr.ldc, pr.out_fp32 ? 4 : 2, pr.M, pr.N, out_row0, col);
          continue;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          // out-of-range rows / columns of the box are clipped by the TMA unit
          if (P.scatter_n > 0) {
            // whole 32-row chunks beyond M (the second CTA of a pair on a short last tile) have no
            // owner: skip them (M is a multiple of 32 in scatter mode)
            if (out_row0 < pr.M) {
              const int owner = out_row0 / P.scatter_rows;
              tma_reduce_add_2d(&P.scatter[owner], slot_ptr(b, 0), pr.scatter_col0 + col,
                                out_row0 - owner * P.scatter_rows);
            }
          } else if (pr.reduce_add) {
            tma_reduce_add_2d(&pr.tma_c, slot_ptr(b, 0), col, out_row0);
          } else {
            tma_store_2d(&pr.tma_c, slot_ptr(b, 0), col, out_row0);
          }
          bulk_commit();
        }
      }
    }
    if (lane == 0) {
      bulk_wait<0>();
      if (P.scatter_n > 0) __threadfence_system();  // the peer reduce-adds are complete and visible
    }
  }

  // pair: neither CTA may leave (or free TMEM) while the leader can still touch the peer
  if constexpr (kPair) cluster_sync_all();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ============================================================================ host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D row-major tensor [outer, inner] with row stride `ld` elements, 128B swizzle.
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint32_t box_inner, uint32_t box_outer, bool fp32 = false) {
  auto enc = get_encode_fn();
  if (!enc) return BTP_ERR_CUDA;
  const uint64_t esz = fp32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? BTP_OK : BTP_ERR_ALIGNMENT;
}

template <int BN, int kSlots, bool kPair>
static int launch(const DevParams& P, int grid, cudaStream_t stream) {
  using C = Cfg<BN, kSlots, kPair>;
  static_assert(C::kSmemBytes <= 232448, "shared memory budget");
  static_assert(2 * C::kStages * 8 + 20 * 8 + 8 <= C::kBarrierBytes, "barrier region");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_kernel<BN, kSlots, kPair>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmemBytes) != cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  if constexpr (!kPair) {
    gemm_kernel<BN, kSlots, kPair><<<grid, kThreads, C::kSmemBytes, stream>>>(P);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, gemm_kernel<BN, kSlots, kPair>, P) != cudaSuccess) return BTP_ERR_CUDA;
  }
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

// N-tile choice: persistent units (CTAs, or CTA pairs) run ceil(tiles / units) waves of tiles
// whose time is ~ BN + a fixed per-tile cost. For CTA pairs that cost is ~192 columns' worth:
// a 256 x 128 pair tile takes ~0.71x (not 0.5x) of a 256 x 256 one (measured on B200,
// tests/gpu_gemm_bn.py), so BN = 256 wins unless its last wave is nearly empty.
static int pick_bn(const btp_gemm_problem* probs, int n, int units, int tile_m, int sig_span) {
  // pair mode stages BN/2 rows of B per CTA; an MN-major B needs whole 64-element chunks, so
  // BN = 192 (96 rows) is single-CTA only
  static const int cands[3] = {256, 192, 128};
  const bool pair = tile_m > kBM;
  int best = sig_span && sig_span % 256 ? 128 : 256;
  long long best_cost = -1;
  for (int c = 0; c < 3; ++c) {
    if (pair && cands[c] == 192) continue;
    if (sig_span && sig_span % cands[c]) continue;  // a sigma tile must not straddle two projections
    const int bn = cands[c];
    long long tiles = 0;
    for (int i = 0; i < n; ++i)
      tiles += (long long)((probs[i].M + tile_m - 1) / tile_m) * ((probs[i].N + bn - 1) / bn) * probs[i].splits;
    const long long waves = (tiles + units - 1) / units;
    const long long cost = waves * (bn + (pair ? 192 : 32));
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = bn; }
  }
  return best;
}

// CTA-pair (cta_group::2) tiles: 0 never, 1 plain / sigma epilogues, 2 also residual epilogues
// (default: with the whole-tile residual staging the pair tiles win there too)
static int g_pair_mode = 2;
// residual epilogues: 3 (default) = by width: narrow outputs (every residual problem N <= 1024,
// e.g. the TP >= 2 o / down up-projections) take the producer-warp pipeline with st.global stores,
// wide ones the whole-tile staging (measured on B200, tests/gpu_gemm_resid_ab.py: [16384 x 512,
// K = 1024] 24.6 -> 19.2 us; [16384 x 2048, K = 512] 37.8 us tile vs 39.4 us pipeline);
// 2 = always the pipeline (kSlots == 5, CTA pairs; single-CTA launches fall back to 1),
// 1 = whole-tile residual staging (kSlots == 4), 0 = per-chunk prefetch (A/B)
static int g_res4 = 3;
// epilogue stores: 0 (default) = TMA bulk-tensor stores, 1 = coalesced st.global from the staging
// chunk for every launch (measured slower for plain epilogues: [16384 x 2048, K = 512] 29.4 ->
// 33.3 us); mode 3 above turns st.global on for the narrow residual launches only
static int g_st_global = 0;

}  // namespace btp

extern "C" int btp_gemm_set_res4(int enable) {
  const int prev = btp::g_res4;
  btp::g_res4 = enable < 0 ? 0 : (enable > 3 ? 3 : enable);
  return prev;
}

extern "C" int btp_gemm_set_st_global(int enable) {
  const int prev = btp::g_st_global;
  btp::g_st_global = enable ? 1 : 0;
  return prev;
}

extern "C" int btp_gemm_set_pair(int enable) {
  const int prev = btp::g_pair_mode;
  btp::g_pair_mode = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
  return prev;
}

namespace btp {

int gemm_launch(const btp_gemm_problem* probs, int n, int bn_hint, int max_ctas, cudaStream_t stream) {
  return gemm_launch_scatter(probs, n, bn_hint, max_ctas, stream, nullptr);
}

int gemm_launch_scatter(const btp_gemm_problem* probs, int n, int bn_hint, int max_ctas, cudaStream_t stream,
                        const ScatterSpec* sc) {
  if (n <= 0 || n > kMaxProblems) return BTP_ERR_DIM;
  if (sc != nullptr) {
    if (sc->n_owners < 1 || sc->n_owners > kMaxOwners || sc->rows_per_owner <= 0 || sc->rows_per_owner % 32 ||
        sc->width <= 0 || sc->width % 8 || sc->ld % 8)
      return BTP_ERR_DIM;
    for (int i = 0; i < n; ++i) {
      const btp_gemm_problem& q = probs[i];
      if (q.c_fp32 || q.splits > 1 || q.reduce_add || q.resid || q.epilogue != kEpiStore) return BTP_ERR_DIM;
      if (q.M != sc->rows_per_owner * sc->n_owners) return BTP_ERR_DIM;
      if (sc->col0[i] < 0 || sc->col0[i] % 8 || sc->col0[i] + q.N > sc->width) return BTP_ERR_DIM;
    }
  }
  for (int i = 0; i < n; ++i) {
    const btp_gemm_problem& q = probs[i];
    if (q.M <= 0 || q.N <= 0 || q.K <= 0) return BTP_ERR_DIM;
    if (q.N % 8 != 0 || q.K % 8 != 0 || q.ldc % 8 != 0) return BTP_ERR_ALIGNMENT;
    if (q.splits < 1) return BTP_ERR_DIM;
    if (q.splits > 1 && !q.c_fp32) return BTP_ERR_DIM;
    if (q.resid && (q.c_fp32 || q.ld_resid % 8)) return BTP_ERR_DIM;
    // split-K accumulates through TMA reduce-add into a zero-initialised fp32 output
    if (q.splits > 1 && !q.reduce_add) return BTP_ERR_DIM;
    if (q.epilogue != kEpiStore && q.epilogue != kEpiSigma && q.epilogue != kEpiSwigluBwd) return BTP_ERR_DIM;
    if ((q.epilogue == kEpiSigma) != (probs[0].epilogue == kEpiSigma)) return BTP_ERR_DIM;  // homogeneous
    if (q.epilogue == kEpiSigma &&
        (q.c_fp32 || q.splits > 1 || q.reduce_add || q.resid || q.b_mn || !q.c2 || q.ldc2 % 8 ||
         q.sigma_half <= 0 || q.sigma_half % 64 || q.N % (2 * q.sigma_half) ||
         q.sigma_half != probs[0].sigma_half))
      return BTP_ERR_DIM;
    if (q.epilogue == kEpiSwigluBwd &&
        (!q.resid || !q.aux2 || !q.c2 || q.c_fp32 || q.splits > 1 || q.reduce_add || q.ld_aux2 % 8 || q.ldc2 % 8))
      return BTP_ERR_DIM;
  }
  int slots = 1;
  for (int i = 0; i < n; ++i) slots = probs[i].epilogue != kEpiStore ? 2 : slots;
  const bool sigma = probs[0].epilogue == kEpiSigma;
  // pair tiles win on plain epilogues, and on residual ones with the whole-tile residual staging
  // (the per-chunk residual prefetch did not gain from them: mode 1 keeps those single-CTA)
  bool any_resid = false;
  for (int i = 0; i < n; ++i) any_resid = any_resid || probs[i].resid != nullptr;
  const bool pair = g_pair_mode && (slots == 1 || sigma) && (!any_resid || g_pair_mode == 2) && num_sms_cached() >= 2;
  const int tile_m = pair ? 2 * kBM : kBM;
  const int units = pair ? num_sms_cached() / 2 : num_sms_cached();
  const int sig_span = probs[0].epilogue == kEpiSigma ? 2 * probs[0].sigma_half : 0;
  int BN = (bn_hint == 128 || bn_hint == 192 || bn_hint == 256) ? bn_hint
                                                                 : pick_bn(probs, n, units, tile_m, sig_span);
  if (pair && BN == 192) BN = 256;
  if (sig_span && (BN == 192 || sig_span % BN)) return BTP_ERR_DIM;
  const int b_rows = pair ? BN / 2 : BN;  // rows of B each CTA stages
  DevParams P;
  memset(&P, 0, sizeof(P));
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    const btp_gemm_problem& q = probs[i];
    DevProblem& d = P.prob[i];
    int rc;
    if (!q.a_mn) rc = make_tmap(&d.tma_a, q.a, q.K, q.M, q.lda, kBK, kBM);
    else         rc = make_tmap(&d.tma_a, q.a, q.M, q.K, q.lda, 64, kBK);
    if (rc) return rc;
    if (q.epilogue == kEpiSigma) rc = make_tmap(&d.tma_b, q.b, q.K, q.N, q.ldb, kBK, BN / 2);
    else if (!q.b_mn) rc = make_tmap(&d.tma_b, q.b, q.K, q.N, q.ldb, kBK, b_rows);
    else         rc = make_tmap(&d.tma_b, q.b, q.N, q.K, q.ldb, 64, kBK);
    if (rc) return rc;
    d.a_mn = q.a_mn != 0;
    d.b_mn = q.b_mn != 0;
    d.idesc = make_idesc_bf16_f32(tile_m, BN, d.a_mn, d.b_mn);
    if (sc == nullptr || q.c != nullptr) {
      rc = make_tmap(&d.tma_c, q.c, q.N, q.M, q.ldc, q.c_fp32 ? 32 : 64, 32, q.c_fp32 != 0);
      if (rc) return rc;
    }
    d.scatter_col0 = sc ? sc->col0[i] : 0;
    if (q.resid) {
      rc = make_tmap(&d.tma_r, q.resid, q.N, q.M, q.ld_resid, 64, 32);
      if (rc) return rc;
    }
    d.epi = q.epilogue;
    d.sig_half = q.epilogue == kEpiSigma ? q.sigma_half : 0;
    if (q.epilogue == kEpiSigma) {
      rc = make_tmap(&d.tma_c2, q.c2, q.N, q.M, q.ldc2, 64, 32);
      if (rc) return rc;
    }
    if (q.epilogue == kEpiSwigluBwd) {
      rc = make_tmap(&d.tma_r2, q.aux2, q.N, q.M, q.ld_aux2, 64, 32);
      if (rc) return rc;
      rc = make_tmap(&d.tma_c2, q.c2, q.N, q.M, q.ldc2, 64, 32);
      if (rc) return rc;
    }
    d.row_scale = q.row_scale;
    d.col_scale = q.col_scale;
    d.c_ptr = reinterpret_cast<char*>(q.c);
    d.ldc = q.ldc;
    d.c2_ptr = reinterpret_cast<char*>(q.c2);
    d.ldc2 = q.ldc2;
    d.resid = reinterpret_cast<const __nv_bfloat16*>(q.resid);
    d.ld_resid = q.ld_resid;
    d.M = q.M; d.N = q.N; d.K = q.K;
    d.m_tiles = (q.M + tile_m - 1) / tile_m;
    d.n_tiles = (q.N + BN - 1) / BN;
    d.k_blocks = (q.K + kBK - 1) / kBK;
    d.kb_per_split = (d.k_blocks + q.splits - 1) / q.splits;
    // splits that would start past the last k-block (e.g. 64 k-blocks in 9 splits of 8) are
    // dropped: an empty split's tile would reduce-add an accumulator no MMA ever wrote
    d.splits = (d.k_blocks + d.kb_per_split - 1) / d.kb_per_split;
    d.out_fp32 = sc != nullptr ? 1 : q.c_fp32;  // scatter: fp32 chunks reduce-added into the owners
    d.reduce_add = q.reduce_add;
    d.alpha = q.alpha == 0.0f ? 1.0f : q.alpha;
    d.tile_start = tiles;
    tiles += d.m_tiles * d.n_tiles * d.splits;
  }
  P.num_problems = n;
  P.total_tiles = tiles;
  P.st_global = g_st_global;
  int max_resid_n = 0;
  for (int i = 0; i < n; ++i)
    if (probs[i].resid) max_resid_n = probs[i].N > max_resid_n ? probs[i].N : max_resid_n;
  if (sc != nullptr) {
    P.scatter_n = sc->n_owners;
    P.scatter_rows = sc->rows_per_owner;
    for (int j = 0; j < sc->n_owners; ++j) {
      const int rc = make_tmap(&P.scatter[j], sc->owners[j], sc->width, sc->rows_per_owner, sc->ld, 32, 32, true);
      if (rc) return rc;
    }
  }
  int grid_units = tiles < units ? tiles : units;
  if (max_ctas > 0 && grid_units > max_ctas) grid_units = max_ctas;
  // residual launches (bf16 outputs only): the whole-tile residual staging layout
  bool res4 = g_res4 && slots == 1 && any_resid && sc == nullptr;
  for (int i = 0; i < n; ++i) res4 = res4 && !probs[i].c_fp32 && !probs[i].reduce_add && probs[i].splits == 1;
  if (pair) {
    const int grid = 2 * grid_units;
    const bool narrow = btp::g_res4 == 3 && max_resid_n <= 1024;
    if (res4 && (btp::g_res4 == 2 || narrow)) {
      if (narrow) P.st_global = 1;
      return BN == 256 ? launch<256, 5, true>(P, grid, stream) : launch<128, 5, true>(P, grid, stream);
    }
    if (res4) return BN == 256 ? launch<256, 4, true>(P, grid, stream) : launch<128, 4, true>(P, grid, stream);
    if (slots == 2) return BN == 256 ? launch<256, 2, true>(P, grid, stream) : launch<128, 2, true>(P, grid, stream);
    if (BN == 256) return launch<256, 1, true>(P, grid, stream);
    return launch<128, 1, true>(P, grid, stream);
  }
  const int grid = grid_units;
  if (res4) {
    if (BN == 256) return launch<256, 4, false>(P, grid, stream);
    if (BN == 192) return launch<192, 4, false>(P, grid, stream);
    return launch<128, 4, false>(P, grid, stream);
  }
  if (slots == 2) {
    if (BN == 256) return launch<256, 2, false>(P, grid, stream);
    if (BN == 192) return launch<192, 2, false>(P, grid, stream);
    return launch<128, 2, false>(P, grid, stream);
  }
  if (BN == 256) return launch<256, 1, false>(P, grid, stream);
  if (BN == 192) return launch<192, 1, false>(P, grid, stream);
  return launch<128, 1, false>(P, grid, stream);
}

}  // namespace btp
