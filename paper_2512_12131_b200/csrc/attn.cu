// Unmasked multi-head attention on tcgen05 / TMEM for sm_100a (bf16 in, fp32 softmax statistics).
//
// The reference runs, per (batch, head), scores = q k^T / sqrt(hd), a row softmax and probs @ v,
// with heads as contiguous feature slices of the [T, heads*hd] activations (model.py:205-230,
// simulator.py:221-233). Here q / k / v / o stay in that [T, width] layout: a head's 128-row tile is
// one TMA box (64 columns = 128 B, 128B swizzle) per 64 head-dim columns, so no transposes or
// per-head copies are ever materialised.
//
// Forward (one CTA per 128-query tile of one (batch, head); two CTAs per SM):
//   w0      TMA producer: Q once, then K_j / V_j into a 2-stage ring
//   w1      TMEM allocator + MMA issuer:  S = Q K_j^T (SS, M128 N128) -> TMEM;
//           after the softmax warps publish P_j:  O += P_j V_j (TS: A = P_j straight from TMEM)
//   w2..w5  softmax: thread i owns query row i == TMEM lane i, so a row's max / sum never leave
//           the thread (no shuffles). exp2 on the MUFU; P_j is written back as packed bf16 over the
//           first 64 columns of S (the MMA reads it as the A operand: no shared-memory round trip).
//           The running max is updated lazily (only when it grows by > 2^8), so the O accumulator
//           in TMEM is rescaled only on those rare tiles; the final 1/l and the log2-domain
//           log-sum-exp (the backward's statistics) are applied in the epilogue.
// The S buffer is single: the next S MMA is issued after P_j is consumed (tcgen05 MMAs of one
// thread execute in order), and the second resident CTA on the SM fills the gap.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "btp_internal.h"
#include "ptx.cuh"

namespace btp {
namespace {

constexpr int kTile = 128;  // query rows per CTA and key/value rows per step

template <int HD, int ST>
struct FwdCfg {
  static constexpr int kTileBytes = kTile * HD * 2;
  static constexpr int kChunks = HD / 64;  // 128-byte-wide TMA boxes per tile
  static constexpr int kTmemCols = (kTile + HD) <= 256 ? 256 : 512;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmem = 1024 + kTileBytes * (1 + 2 * ST) + kBarBytes;
  static constexpr int kThreads = 192;
};

struct FwdParams {
  CUtensorMap tq, tk, tv;
  __nv_bfloat16* o;
  long long ldo;
  float* lse;  // [b, h, s]: log2-domain log-sum-exp of the scaled scores (m + log2 l)
  int s, h, n_kv;
  float c;  // log2(e) / sqrt(hd)
  long long* trace;  // optional clock64 stamps of CTA (0, 0, 0), [n_kv][16] (pipeline diagnostics)
  int dry;           // diagnostics (split-row kernels, wrong results): softmax warps only do the handshakes
};

template <int HD, int ST, int kPoly>
__global__ void __launch_bounds__(192, 2) attn_fwd_kernel(const __grid_constant__ FwdParams P) {
  using C = FwdCfg<HD, ST>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::kTileBytes;
  uint8_t* sV = sK + ST * C::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ST * C::kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_full = kv_empty + ST;
  uint64_t* p_full = s_full + 1;
  uint64_t* o_bar = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 1);

  const int qt = blockIdx.x, head = blockIdx.y, bi = blockIdx.z;
  const int row0 = bi * P.s + qt * kTile;
  const int kv0 = bi * P.s;
  const int col0 = head * HD;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < ST; ++s) {
        mbar_init(&kv_full[s], 1);
        mbar_init(&kv_empty[s], 1);
      }
      mbar_init(s_full, 1);
      mbar_init(p_full, 4);
      mbar_init(o_bar, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + kTile;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, C::kTileBytes);
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c) tma_load_2d(sQ + c * kTile * 128, &P.tq, q_full, col0 + 64 * c, row0);
      for (int j = 0; j < P.n_kv; ++j) {
        const int st = j % ST;
        const uint32_t ph = (j / ST) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::kTileBytes);
        uint8_t* k_dst = sK + st * C::kTileBytes;
        uint8_t* v_dst = sV + st * C::kTileBytes;
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(k_dst + c * kTile * 128, &P.tk, &kv_full[st], col0 + 64 * c, kv0 + j * kTile);
          tma_load_2d(v_dst + c * kTile * 128, &P.tv, &kv_full[st], col0 + 64 * c, kv0 + j * kTile);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16_f32(kTile, kTile, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16_f32(kTile, HD, false, true);
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t q_base = smem_u32(sQ);
    for (int j = 0; j < P.n_kv; ++j) {
      const int st = j % ST;
      const uint32_t ph = (j / ST) & 1;
      mbar_wait(&kv_full[st], ph);
      tc_fence_after();
      const uint32_t k_base = smem_u32(sK + st * C::kTileBytes);
      const uint32_t v_base = smem_u32(sV + st * C::kTileBytes);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * kTile * 128 + (k & 3) * 32;  // K-major: 32 B per 16 elements
          umma_bf16(tS, make_sw128_desc(q_base + off, 16, 1024), make_sw128_desc(k_base + off, 16, 1024), idesc_s,
                    k > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
      }
      __syncwarp();
      mbar_wait(p_full, j & 1);
      tc_fence_after();
      if (elect_one()) {
        // P_j (bf16 pairs in S columns [0, 64)) x V_j: V is MN-major ([kv, hd] rows of 128 B);
        // 16 kv rows = 2 KB per K step, 64-column chunks kTile * 128 B apart (LBO).
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k) {
          umma_bf16_ts(tO, tS + k * 8, make_sw128_desc(v_base + k * 2048, kTile * 128, 1024), idesc_o,
                       (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&kv_empty[st]);
        umma_commit(o_bar);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- softmax (warps 2..5)
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const float c = P.c;
    float m_used = 0.f, l = 0.f;
    for (int j = 0; j < P.n_kv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      uint32_t s[128];
      tmem_ld_32x32b_x64(tS + lane_addr, *reinterpret_cast<uint32_t(*)[64]>(&s[0]));
      tmem_ld_32x32b_x64(tS + lane_addr + 64, *reinterpret_cast<uint32_t(*)[64]>(&s[64]));
      tmem_ld_wait();
      float mx[4] = {__uint_as_float(s[0]), __uint_as_float(s[1]), __uint_as_float(s[2]), __uint_as_float(s[3])};
#pragma unroll
      for (int i = 4; i < 128; i += 8) {
        mx[0] = fmax3(mx[0], __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
        mx[1] = fmax3(mx[1], __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
        if (i + 4 < 128) {
          mx[2] = fmax3(mx[2], __uint_as_float(s[i + 4]), __uint_as_float(s[i + 5]));
          mx[3] = fmax3(mx[3], __uint_as_float(s[i + 6]), __uint_as_float(s[i + 7]));
        }
      }
      const float m_new = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * c;
      if (j == 0) {
        m_used = m_new;
      } else {
        const bool need = m_new > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          // rescale this row's O accumulator once PV_{j-1} has landed
          mbar_wait(o_bar, (j - 1) & 1);
          tc_fence_after();
          const float alpha = need ? ex2_approx(m_used - m_new) : 1.f;
#pragma unroll
          for (int cc = 0; cc < HD / 32; ++cc) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + lane_addr + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(tO + lane_addr + cc * 32, o);
          }
          tmem_st_wait();
          if (need) {
            l *= alpha;
            m_used = m_new;
          }
        }
      }
      // exp2 on the MUFU, except every kPoly-th pair on the FMA pipe (ex2_poly2): the MUFU's 16 / clk / SM
      // is this loop's bound
      float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      const float2 c2 = make_float2(c, c), nm = make_float2(-m_used, -m_used);
      // P pair i is packed into s[i] (s[2i], s[2i+1] are consumed by then): no second 64-register array
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nm);
        float2 e;
        if (kPoly > 0 && (i % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
          e = ex2_poly2(x);
        } else {
          e.x = ex2_approx(x.x);
          e.y = ex2_approx(x.y);
        }
        if (i & 1) l2b = fadd2(l2b, e);
        else l2a = fadd2(l2a, e);
        s[i] = pack_bf16(e.x, e.y);
      }
      l += (l2a.x + l2a.y) + (l2b.x + l2b.y);
      tmem_st_32x32b_x32(tS + lane_addr, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
      tmem_st_32x32b_x32(tS + lane_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    mbar_wait(o_bar, (P.n_kv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = P.o + (long long)(row0 + row) * P.ldo + col0;
#pragma unroll
    for (int cc = 0; cc < HD / 32; ++cc) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tO + lane_addr + cc * 32, o);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_global_v4(orow + cc * 32 + v * 8, make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
    }
    P.lse[((long long)bi * P.h + head) * P.s + qt * kTile + row] = m_used + __log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------- forward, split rows
// The kernel above alternates, per query tile, softmax and the PV + next-S MMAs on one S buffer, so
// each CTA's softmax waits ~800 tensor cycles per key tile (2 CTAs / SM only partly hide it). This one
// (one CTA / SM, 512 TMEM columns):
//   * double-buffers S (columns 0 / 128): S_{j+1} is computed while the softmax works on S_j;
//   * splits every query row's 128 keys over two warps (group g = keys [64g, 64g + 64)), each with its
//     OWN running max m_g, sum l_g and O accumulator O_g (columns 256 + g*hd): no cross-warp exchange
//     inside the loop, 8 softmax warps (two per scheduler); PV is two K = 64 MMA chains (O_g += P_g V_g);
//   * combines once at the end: O = (O_0 2^(m_0-m) + O_1 2^(m_1-m)) / (l_0 2^(m_0-m) + l_1 2^(m_1-m)).
// kSplit key groups per row (2, or 4 at hd 64: 2 S buffers + 4 O accumulators fill the 512 columns).
// kSBuf = 1: one S buffer (S_{j+1} issued after PV_j, like attn_fwd_kernel) so that at hd 64 / kSplit 2
// the CTA needs 256 TMEM columns and two CTAs share an SM (16 softmax warps per SM).
// kQT = 2: two 128-row query tiles per CTA share every K / V tile (half the K / V traffic from L2 per
// query row); each has its own S buffer, softmax warps and O accumulators, and the two softmax groups
// ping-pong with the tensor core (S / PV of one tile run while the other's softmax does).
template <int HD, int ST, int kSplit, int kSBuf = 2, int kQT = 1>
struct Fwd2Cfg {
  static constexpr int kTileBytes = kTile * HD * 2;
  static constexpr int kChunks = HD / 64;
  static constexpr int kKG = kTile / kSplit;              // keys per group
  static constexpr int kNS = kQT * kSBuf;                 // S buffers
  static constexpr int kMlBytes = kQT * kSplit * 2 * kTile * 4;  // (m, l) per tile, group and row
  static constexpr int kBarBytes = 256;
  static constexpr int kSmem = 1024 + kTileBytes * (kQT + 2 * ST) + kMlBytes + kBarBytes;
  static constexpr int kSoftWarps = 4 * kSplit * kQT;
  static constexpr int kThreads = 64 + 32 * kSoftWarps;
  static constexpr uint32_t tO = 128 * kNS;  // O_(u,g) at tO + (u * kSplit + g) * HD
  static constexpr uint32_t kCols = (tO + kQT * kSplit * HD <= 256) ? 256 : 512;
  static constexpr int kCtasPerSm = kCols == 256 ? 2 : 1;
  static_assert(tO + kQT * kSplit * HD <= 512, "TMEM budget");
  static_assert(kQT == 1 || kSBuf == 1, "two query tiles use one S buffer each");
};

template <int HD, int ST, int kPoly, int kSplit, int kSBuf, int kQT>
__global__ void __launch_bounds__(Fwd2Cfg<HD, ST, kSplit, kSBuf, kQT>::kThreads,
                                  Fwd2Cfg<HD, ST, kSplit, kSBuf, kQT>::kCtasPerSm)
    attn_fwd2_kernel(const __grid_constant__ FwdParams P) {
  using C = Fwd2Cfg<HD, ST, kSplit, kSBuf, kQT>;
  constexpr int kKG = C::kKG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kQT * C::kTileBytes;
  uint8_t* sV = sK + ST * C::kTileBytes;
  float* sML = reinterpret_cast<float*>(sV + ST * C::kTileBytes);  // [kSplit groups][m | l][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sML) + C::kMlBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_full = kv_empty + ST;  // [kNS]
  uint64_t* p_full = s_full + 2 * kQT;  // [kNS]
  uint64_t* o_bar = p_full + 2 * kQT;   // [kQT], one phase per PV
  uint64_t* o_final = o_bar + kQT;      // [kQT]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + kQT);

  const int qt = blockIdx.x, head = blockIdx.y, bi = blockIdx.z;
  const int row0 = bi * P.s + qt * kTile * kQT;
  const int kv0 = bi * P.s;
  const int col0 = head * HD;
  const int n = P.n_kv;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  long long* const tr = (qt == 0 && head == 0 && bi == 0) ? P.trace : nullptr;
#define FSTAMP(jj, e)                                               \
  do {                                                              \
    if (tr != nullptr && lane == 0) tr[(jj) * 16 + (e)] = clock64(); \
  } while (0)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < ST; ++s) {
        mbar_init(&kv_full[s], 1);
        mbar_init(&kv_empty[s], 1);
      }
      for (int b = 0; b < C::kNS; ++b) {
        mbar_init(&s_full[b], 1);
        mbar_init(&p_full[b], 4 * kSplit);
      }
      for (int u = 0; u < kQT; ++u) {
        mbar_init(&o_bar[u], 1);
        mbar_init(&o_final[u], 1);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<C::kCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, kQT * C::kTileBytes);
#pragma unroll
      for (int u = 0; u < kQT; ++u)
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_2d(sQ + u * C::kTileBytes + c * kTile * 128, &P.tq, q_full, col0 + 64 * c, row0 + u * kTile);
      for (int j = 0; j < n; ++j) {
        const int st = j % ST;
        mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(sK + st * C::kTileBytes + c * kTile * 128, &P.tk, &kv_full[st], col0 + 64 * c, kv0 + j * kTile);
          tma_load_2d(sV + st * C::kTileBytes + c * kTile * 128, &P.tv, &kv_full[st], col0 + 64 * c, kv0 + j * kTile);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16_f32(kTile, kTile, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16_f32(kTile, HD, false, true);
    auto issue_s = [&](int u, int j) {  // S_(u,j) = Q_u K_j^T into buffer u * kSBuf + j % kSBuf
      const int st = j % ST;
      mbar_wait(&kv_full[st], (j / ST) & 1);
      tc_fence_after();
      const uint32_t k_base = smem_u32(sK + st * C::kTileBytes);
      const uint32_t q_base = smem_u32(sQ + u * C::kTileBytes);
      const int b = u * kSBuf + j % kSBuf;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * kTile * 128 + (k & 3) * 32;
          umma_bf16(tmem + b * 128, make_sw128_desc(q_base + off, 16, 1024),
                    make_sw128_desc(k_base + off, 16, 1024), idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[b]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    tc_fence_after();
    for (int u = 0; u < kQT; ++u) issue_s(u, 0);
    if (kSBuf == 2 && n > 1) issue_s(0, 1);
    for (int j = 0; j < n; ++j) {
      const int st = j % ST;
      const uint32_t v_base = smem_u32(sV + st * C::kTileBytes);
#pragma unroll
      for (int u = 0; u < kQT; ++u) {
        const int b = u * kSBuf + j % kSBuf;
        mbar_wait(&p_full[b], (j / kSBuf) & 1);
        if (u == 0) FSTAMP(j, 8);
        tc_fence_after();
        if (elect_one()) {
          // O_(u,g) += P_g V[kKG g, kKG (g + 1)): A = P_g (bf16 pairs at S columns kKG g ..), B = V (MN-major)
#pragma unroll
          for (int g = 0; g < kSplit; ++g) {
#pragma unroll
            for (int k = 0; k < kKG / 16; ++k)
              umma_bf16_ts(tmem + C::tO + (u * kSplit + g) * HD, tmem + b * 128 + g * kKG + k * 8,
                           make_sw128_desc(v_base + (g * kKG + 16 * k) * 128, kTile * 128, 1024), idesc_o,
                           (j > 0 || k > 0) ? 1u : 0u);
          }
          if (u == kQT - 1) umma_commit(&kv_empty[st]);
          umma_commit(&o_bar[u]);
          if (j == n - 1) umma_commit(&o_final[u]);
        }
        __syncwarp();
        if (u == 0) FSTAMP(j, 9);
        if (j + kSBuf < n) issue_s(u, j + kSBuf);  // into buffer b, which P_(u,j) (just consumed) aliased
        if (u == 0) FSTAMP(j, 10);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax warps 2 .. 2 + 4 kSplit
    const uint32_t sw = (warp - 2) >> 2;
    const uint32_t g = sw % kSplit;  // key group
    const uint32_t u = sw / kSplit;  // query tile
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const uint32_t tOg = tmem + C::tO + (u * kSplit + g) * HD + lane_addr;
    const float c = P.c;
    float m_used = 0.f, l = 0.f;
    for (int j = 0; j < n; ++j) {
      const int b = u * kSBuf + j % kSBuf;
      const uint32_t tSg = tmem + b * 128 + g * kKG + lane_addr;
      mbar_wait(&s_full[b], (j / kSBuf) & 1);
      if (q4 == 2 && u == 0) FSTAMP(j, 4 * g);
      tc_fence_after();
      if (P.dry) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        continue;
      }
      // two passes over the group's kKG columns in 32-column chunks (registers: one chunk at a time;
      // TMEM reads are cheap): max, then exp2 / sum / bf16 pairs written back over the consumed columns
      float mx[4] = {-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f};
#pragma unroll
      for (int ch = 0; ch < kKG / 32; ++ch) {
        uint32_t s[32];
        tmem_ld_32x32b_x32(tSg + ch * 32, s);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          mx[0] = fmax3(mx[0], __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
          mx[1] = fmax3(mx[1], __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
          mx[2] = fmax3(mx[2], __uint_as_float(s[i + 4]), __uint_as_float(s[i + 5]));
          mx[3] = fmax3(mx[3], __uint_as_float(s[i + 6]), __uint_as_float(s[i + 7]));
        }
      }
      const float m_new = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * c;
      if (q4 == 2 && u == 0) FSTAMP(j, 4 * g + 1);
      if (j == 0) {
        m_used = m_new;
      } else {
        const bool need = m_new > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          // O_g must hold PV_{j-1} before it is rescaled (S_j was issued after PV_{j-kSBuf}: the barrier
          // is at phase j-1 or j, so the parity wait is unambiguous)
          mbar_wait(&o_bar[u], (j - 1) & 1);
          tc_fence_after();
          const float alpha = need ? ex2_approx(m_used - m_new) : 1.f;
#pragma unroll
          for (int cc = 0; cc < HD / 32; ++cc) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tOg + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(tOg + cc * 32, o);
          }
          tmem_st_wait();
          if (need) {
            l *= alpha;
            m_used = m_new;
          }
        }
      }
      float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      const float2 c2 = make_float2(c, c), nm = make_float2(-m_used, -m_used);
#pragma unroll
      for (int ch = 0; ch < kKG / 32; ++ch) {
        uint32_t s[32];
        tmem_ld_32x32b_x32(tSg + ch * 32, s);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nm);
          float2 e;
          if (kPoly > 0 && ((ch * 16 + i) % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
            e = ex2_poly2(x);
          } else {
            e.x = ex2_approx(x.x);
            e.y = ex2_approx(x.y);
          }
          if (i & 1) l2b = fadd2(l2b, e);
          else l2a = fadd2(l2a, e);
          s[i] = pack_bf16(e.x, e.y);
        }
        tmem_st_32x32b_x16(tSg + ch * 16, *reinterpret_cast<uint32_t(*)[16]>(&s[0]));
      }
      l += (l2a.x + l2a.y) + (l2b.x + l2b.y);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      if (q4 == 2 && u == 0) FSTAMP(j, 4 * g + 2);
    }
    // ---------------------------------------------------------------- epilogue: combine the groups
    float* ml = sML + u * (kSplit * 2 * kTile);
    ml[(g * 2 + 0) * kTile + row] = m_used;
    ml[(g * 2 + 1) * kTile + row] = l;
    named_bar_sync(1 + u, 32 * 4 * kSplit);
    float mg[kSplit], lg[kSplit];
    float m = -3.0e38f;
#pragma unroll
    for (int x = 0; x < kSplit; ++x) {
      mg[x] = ml[(x * 2) * kTile + row];
      lg[x] = ml[(x * 2 + 1) * kTile + row];
      m = fmaxf(m, mg[x]);
    }
    float L = 0.f;
#pragma unroll
    for (int x = 0; x < kSplit; ++x) {
      mg[x] = ex2_approx(mg[x] - m);  // group weight before normalisation
      L = fmaf(lg[x], mg[x], L);
    }
    const float inv = 1.f / L;
    mbar_wait(&o_final[u], 0);
    tc_fence_after();
    __nv_bfloat16* orow = P.o + (long long)(row0 + u * kTile + row) * P.ldo + col0;
    constexpr int kOC = HD / kSplit;  // output columns of this warp: [g kOC, (g + 1) kOC)
#pragma unroll
    for (int cc = 0; cc < kOC / 16; ++cc) {
      const int oc = g * kOC + cc * 16;
      float acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = 0.f;
#pragma unroll
      for (int x = 0; x < kSplit; ++x) {
        uint32_t ox[16];
        tmem_ld_32x32b_x16(tmem + C::tO + (u * kSplit + x) * HD + oc + lane_addr, ox);
        tmem_ld_wait();
        const float w = mg[x] * inv;
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(__uint_as_float(ox[i]), w, acc[i]);
      }
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] = pack_bf16(acc[2 * i], acc[2 * i + 1]);
      st_global_v4(orow + oc, make_uint4(pk[0], pk[1], pk[2], pk[3]));
      st_global_v4(orow + oc + 8, make_uint4(pk[4], pk[5], pk[6], pk[7]));
    }
    if (g == 0) P.lse[((long long)bi * P.h + head) * P.s + (qt * kQT + u) * kTile + row] = m + __log2f(L);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
#undef FSTAMP
}

// ---------------------------------------------------------------------------- forward, P apart from S
// hd 64. In the kernels above P_j is written over S_j, so S_{j+1} of a query tile can only be issued
// after PV_j has read P_j: per tile the chain S MMA -> softmax -> PV MMA -> next S MMA is serial, and
// the traces show the softmax warps waiting on it (~1580 cycles per (query, key) tile against the
// MUFU's 1024). Here each query tile has its own P columns, so the softmax releases S_j as soon as
// it has pulled the row into registers and S_{j+1} runs on the tensor core underneath softmax j:
//   TMEM (512 columns): S_u at 128 u, P_u (bf16 pairs) at 256 + 64 u, O_u at 384 + 64 u, u = 0, 1
//   w0 TMA (Q_0, Q_1 once; K_j / V_j ring of ST stages), w1 MMA, w2..w9 softmax (query tile u =
//   (w - 2) / 4; thread = query row = TMEM lane, all 128 keys of the tile in registers).
// MMA issue order per key tile j and query tile u: PV_(u,j) once P_(u,j) is published, then
// S_(u,j+2) once softmax (u, j+1) has released S_u (S_(u,0), S_(u,1) before the loop). The two query
// tiles' softmax groups share every K / V tile and keep each scheduler's MUFU fed in turn.
// Measured (profiles/attention/README.md): S never gates the softmax any more; the loop runs at the
// exp2 rate two warps per scheduler reach (scripts/microbench/softmax_rate.cu), ~4 % ahead of the
// two-query-tile kernel above at the bench shape; opt-in, btp_attn_tune(1, 5) / (1, 6) split rows.
// kHalves = 2: every query row's 128 keys are split over two warps (64 each: 16 softmax warps, four
// per scheduler, which is what keeps the MUFU busy - scripts/microbench/softmax_rate.cu); the pair
// shares O_u and P_u (each writes its 32 P columns), exchanges its row maxima through shared memory
// every key tile (so both halves take identical lazy-rescale decisions), and sums l in the epilogue.
template <int ST, int kHalves>
struct Fwd3Cfg {
  static constexpr int kTileBytes = kTile * 64 * 2;
  static constexpr int kBarBytes = 256;
  static constexpr int kXBytes = kHalves == 2 ? 2 * 2 * 2 * kTile * 4 : 0;  // [j & 1][u][half][row] maxima
  static constexpr int kSmem = 1024 + kTileBytes * (2 + 2 * ST) + kXBytes + kBarBytes;
  static constexpr int kSoftWarps = 8 * kHalves;
  static constexpr int kThreads = 64 + 32 * kSoftWarps;
  static constexpr int kKW = kTile / kHalves;  // keys per softmax warp
  static constexpr uint32_t tP = 256, tO = 384;
};

template <int ST, int kPoly, int kHalves>
__global__ void __launch_bounds__(Fwd3Cfg<ST, kHalves>::kThreads, 1)
    attn_fwd3_kernel(const __grid_constant__ FwdParams P) {
  using C = Fwd3Cfg<ST, kHalves>;
  constexpr int kKW = C::kKW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + 2 * C::kTileBytes;
  uint8_t* sV = sK + ST * C::kTileBytes;
  float* sX = reinterpret_cast<float*>(sV + ST * C::kTileBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ST * C::kTileBytes + C::kXBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_full = kv_empty + ST;  // [2]
  uint64_t* s_free = s_full + 2;     // [2]
  uint64_t* p_full = s_free + 2;     // [2]
  uint64_t* o_bar = p_full + 2;      // [2], one phase per PV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 2);

  const int qt = blockIdx.x, head = blockIdx.y, bi = blockIdx.z;
  const int row0 = bi * P.s + qt * 2 * kTile;
  const int kv0 = bi * P.s;
  const int col0 = head * 64;
  const int n = P.n_kv;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  long long* const tr = (qt == 0 && head == 0 && bi == 0) ? P.trace : nullptr;
#define FSTAMP(jj, e)                                               \
  do {                                                              \
    if (tr != nullptr && lane == 0) tr[(jj) * 16 + (e)] = clock64(); \
  } while (0)

  if (warp == 1) FSTAMP(0, 12);  // CTA start
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < ST; ++s) {
        mbar_init(&kv_full[s], 1);
        mbar_init(&kv_empty[s], 1);
      }
      for (int u = 0; u < 2; ++u) {
        mbar_init(&s_full[u], 1);
        mbar_init(&s_free[u], 4 * kHalves);
        mbar_init(&p_full[u], 4 * kHalves);
        mbar_init(&o_bar[u], 1);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 1) FSTAMP(0, 13);  // barriers + TMEM ready

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, 2 * C::kTileBytes);
      tma_load_2d(sQ, &P.tq, q_full, col0, row0);
      tma_load_2d(sQ + C::kTileBytes, &P.tq, q_full, col0, row0 + kTile);
      for (int j = 0; j < n; ++j) {
        const int st = j % ST;
        mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::kTileBytes);
        tma_load_2d(sK + st * C::kTileBytes, &P.tk, &kv_full[st], col0, kv0 + j * kTile);
        tma_load_2d(sV + st * C::kTileBytes, &P.tv, &kv_full[st], col0, kv0 + j * kTile);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16_f32(kTile, kTile, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16_f32(kTile, 64, false, true);
    auto issue_s = [&](int u, int j) {  // S_(u,j) = Q_u K_j^T
      const int st = j % ST;
      mbar_wait(&kv_full[st], (j / ST) & 1);
      tc_fence_after();
      const uint32_t k_base = smem_u32(sK + st * C::kTileBytes);
      const uint32_t q_base = smem_u32(sQ + u * C::kTileBytes);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem + u * 128, make_sw128_desc(q_base + k * 32, 16, 1024),
                    make_sw128_desc(k_base + k * 32, 16, 1024), idesc_s, k > 0 ? 1u : 0u);
        umma_commit(&s_full[u]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int u, int j) {  // O_u += P_(u,j) V_j
      const int st = j % ST;
      mbar_wait(&p_full[u], j & 1);
      FSTAMP(j, 8 + 2 * u);
      tc_fence_after();
      const uint32_t v_base = smem_u32(sV + st * C::kTileBytes);
      if (elect_one()) {
        // A = P_u (bf16 pairs, 8 columns per 16 keys), B = V (MN-major, 2 KB per 16 keys)
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + C::tO + u * 64, tmem + C::tP + u * 64 + k * 8,
                       make_sw128_desc(v_base + k * 2048, kTile * 128, 1024), idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        if (u == 1) umma_commit(&kv_empty[st]);
        umma_commit(&o_bar[u]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    if (n > 1) {
      for (int u = 0; u < 2; ++u) {
        mbar_wait(&s_free[u], 0);
        issue_s(u, 1);
      }
    }
    for (int j = 0; j < n; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        issue_pv(u, j);
        if (j + 2 < n) {
          mbar_wait(&s_free[u], (j + 1) & 1);
          issue_s(u, j + 2);
          FSTAMP(j, 9 + 2 * u);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax warps 2 .. 2 + 8 kHalves
    const uint32_t u = (warp - 2) / (4 * kHalves);
    const uint32_t hf = ((warp - 2) >> 2) % kHalves;  // key half of the row
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const uint32_t tS = tmem + u * 128 + hf * kKW + lane_addr;
    const uint32_t tPu = tmem + C::tP + u * 64 + hf * (kKW / 2) + lane_addr;
    const uint32_t tOu = tmem + C::tO + u * 64 + lane_addr;
    constexpr int kOW = 64 / kHalves;  // O columns this warp rescales / writes: [hf kOW, (hf + 1) kOW)
    // the two warps of a row pair (kHalves = 2) meet on named barrier 1 + 4 u + q4 (64 threads)
    auto pair_max = [&](int j, float m) {
      if (kHalves == 1) return m;
      float* x = sX + (((j & 1) * 2 + u) * 2) * kTile;
      x[hf * kTile + row] = m;
      named_bar_sync(1 + 4 * u + q4, 64);
      return fmaxf(m, x[(hf ^ 1) * kTile + row]);
    };
    const float c = P.c;
    float m_used = 0.f, l = 0.f;
    auto row_max = [&](const uint32_t* v, int cnt, float m) {
      float mx[2] = {m, m};
#pragma unroll
      for (int i = 0; i < cnt; i += 4) {
        mx[0] = fmax3(mx[0], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        mx[1] = fmax3(mx[1], __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
      }
      return fmaxf(mx[0], mx[1]);
    };
    // rescale O_u / l when the row max grew by > 2^8 (lazy): O_u must hold PV_(u,j-1) first
    auto rescale = [&](int j, float m_new) {
      if (j == 0) {
        m_used = m_new;
        return;
      }
      const bool need = m_new > m_used + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        mbar_wait(&o_bar[u], (j - 1) & 1);  // completed PVs: j - 1 or j
        tc_fence_after();
        const float alpha = need ? ex2_approx(m_used - m_new) : 1.f;
#pragma unroll
        for (int cc = 0; cc < kOW / 16; ++cc) {
          uint32_t o[16];
          tmem_ld_32x32b_x16(tOu + hf * kOW + cc * 16, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st_32x32b_x16(tOu + hf * kOW + cc * 16, o);
        }
        tmem_st_wait();
        if (need) {
          l *= alpha;
          m_used = m_new;
        }
      }
    };
    const bool stamp = q4 == 2 && hf == 0;
    uint32_t s[kKW];
    for (int j = 0; j < n; ++j) {
      mbar_wait(&s_full[u], j & 1);
      tc_fence_after();
      if (stamp) FSTAMP(j, 4 * u + 0);
#pragma unroll
      for (int cc = 0; cc < kKW / 64; ++cc)
        tmem_ld_32x32b_x64(tS + cc * 64, *reinterpret_cast<uint32_t(*)[64]>(&s[cc * 64]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[u]);  // S_u may now take S_(u,j+1)
      rescale(j, pair_max(j, row_max(s, kKW, -3.0e38f)) * c);
      if (stamp) FSTAMP(j, 4 * u + 1);
      float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
      const float2 c2 = make_float2(c, c), nm = make_float2(-m_used, -m_used);
#pragma unroll
      for (int i = 0; i < kKW / 2; ++i) {  // P pair i packed into s[i] (s[2i], s[2i+1] are consumed by then)
        const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nm);
        float2 e;
        if (kPoly > 0 && (i % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
          e = ex2_poly2(x);
        } else {
          e.x = ex2_approx(x.x);
          e.y = ex2_approx(x.y);
        }
        if (i & 1) l2b = fadd2(l2b, e);
        else l2a = fadd2(l2a, e);
        s[i] = pack_bf16(e.x, e.y);
      }
      l += (l2a.x + l2a.y) + (l2b.x + l2b.y);
      if (j > 0) {
        mbar_wait(&o_bar[u], (j - 1) & 1);  // PV_(u,j-1) has read P_u
        tc_fence_after();
      }
      if (stamp) FSTAMP(j, 4 * u + 3);
#pragma unroll
      for (int cc = 0; cc < kKW / 64; ++cc)
        tmem_st_32x32b_x32(tPu + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[cc * 32]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[u]);
      if (stamp) FSTAMP(j, 4 * u + 2);
    }
    if (kHalves == 2) {  // l of the whole row: the two halves' partial sums (same reference max)
      float* x = sX + (((n & 1) * 2 + u) * 2) * kTile;
      x[hf * kTile + row] = l;
      named_bar_sync(1 + 4 * u + q4, 64);
      l += x[(hf ^ 1) * kTile + row];
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    mbar_wait(&o_bar[u], (n - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = P.o + (long long)(row0 + u * kTile + row) * P.ldo + col0 + hf * kOW;
#pragma unroll
    for (int cc = 0; cc < kOW / 32; ++cc) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tOu + hf * kOW + cc * 32, o);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_global_v4(orow + cc * 32 + v * 8, make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
    }
    if (hf == 0) P.lse[((long long)bi * P.h + head) * P.s + (qt * 2 + u) * kTile + row] = m_used + __log2f(l);
    if (stamp && u == 0) FSTAMP(0, 14);  // epilogue stored
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
    FSTAMP(0, 15);  // CTA done
  }
#undef FSTAMP
}

// ============================================================================ backward
//
// One CTA per 128-row key/value tile of one (batch, head) (one CTA per SM: 512 TMEM columns);
// the CTA walks every 128-row query tile i:
//   [1] S^T_i  = K Q_i^T        (SS)  -> tS     lane = key row n, column = query m
//   [2] dP^T_i = V dO_i^T       (SS)  -> tdP
//   compute warps: P^T = exp2(S^T c - lse[m]) -> bf16 over tS;  dS^T = P^T (dP^T - D[m]) -> bf16 over
//                  tdP and, MN-major 128B-swizzled, into shared memory (the A operand of [5])
//   [3] dV += P^T_i dO_i        (TS: A = P^T from TMEM)
//   [4] dK += dS^T_i Q_i        (TS: A = dS^T from TMEM)
//   [5] dQ_i = dS_i K           (SS: A = dS from shared memory) -> tdQ; four reduce warps add it
//       into the fp32 dQ accumulator in global memory (vector red.add; summed over the key tiles)
// dK / dV stay in TMEM for the whole walk and are written once (dK scaled by 1/sqrt(hd)).
// MMA issue order [1]_0 [2]_0 | [3]_i [1]_{i+1} [4]_i [5]_i [2]_{i+1} | ... lets the tensor core run
// the next tile's S^T while the compute warps form dS of this one (tcgen05 MMAs of one thread
// execute in issue order, which is what makes the TMEM aliasing safe).
// D = rowsum(dO o O) and the zeroed dQ accumulator come from attn_bwd_prep; attn_bwd_dq converts the
// accumulator to bf16 with the 1/sqrt(hd) scale.
template <int HD, int ST>
struct BwdCfg {
  static constexpr int kTileBytes = kTile * HD * 2;
  static constexpr int kChunks = HD / 64;
  static constexpr int kDsBytes = kTile * kTile * 2;  // dS (bf16) MN-major: 2 chunks of 64 queries
  static constexpr int kStageBytes = 2 * kTileBytes + 2 * kTile * 4;  // Q, dO, lse, D
  static constexpr int kBarBytes = 128;
  static constexpr int kBody = 2 * kTileBytes + ST * kStageBytes + kDsBytes + kBarBytes;
  // 1 KB of slack for aligning the dynamic window to the 128B-swizzle atom, when it fits; without
  // it (hd 128, two stages) the kernel checks that the window is already 1 KB aligned.
  static constexpr int kSlack = (kBody + 1024 <= 232448) ? 1024 : 0;
  static constexpr int kSmem = kSlack + kBody;
  static constexpr int kThreads = 448;
  // TMEM columns
  static constexpr uint32_t tS = 0, tdP = 128, tdV = 256, tdK = 256 + HD;
  static constexpr uint32_t tdQ = (HD == 64) ? 384 : tdP;  // hd 128: dQ reuses the dP / dS columns
};

struct BwdParams {
  CUtensorMap tq, tk, tv, tdo;
  CUtensorMap tdq;  // fp32 dq_acc, 32-column x 128-row boxes, 128B swizzle (hd-64 kernel's TMA reduce)
  const float* lse;  // [b, h, s] log2 domain (attn_fwd)
  const float* D;    // [b, h, s] rowsum(dO o O)
  float* dq_acc;     // fp32 [b*s, ldacc]
  long long ldacc;
  __nv_bfloat16* dk;
  long long lddk;
  __nv_bfloat16* dv;
  long long lddv;
  int s, h, n_q;
  float c;         // log2(e) / sqrt(hd)
  float dk_scale;  // 1 / sqrt(hd)
  long long* trace;  // optional: per-iteration clock64 stamps of CTA (0, 0, 0) (pipeline diagnostics)
  int dry;           // diagnostics (split-role kernel): 1 = P / dS / reduce warps only do the handshakes
  int diag;          // diagnostics (split-role kernel, wrong results): bit0 no dS st.shared, bit1 no proxy
                     // fence after them, bit2 no lse / D shared loads
  int n_items;       // hd-64 kernel: key tiles x heads x batch (work items, walked persistently)
};

#define BTP_STAMP64(e)                                                                            \
  do {                                                                                            \
    if constexpr (kTrace) {                                                                       \
      if (tr != nullptr && lane == 0) tr[i * 16 + (e)] = clock64();                               \
    }                                                                                             \
  } while (0)

#define BTP_STAMP(e)                                                                              \
  do {                                                                                            \
    if (tr != nullptr && lane == 0) tr[i * 16 + (e)] = clock64();                                 \
  } while (0)

__device__ __forceinline__ void red_add_v4(float* ptr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

template <int HD, int ST>
__global__ void __launch_bounds__(448, 1) attn_bwd_kernel(const __grid_constant__ BwdParams P) {
  using C = BwdCfg<HD, ST>;
  static_assert(ST >= 2, "S^T of the next query tile is issued before this tile's dK MMA releases its stage");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if constexpr (C::kSlack == 0) {
    if (smem_u32(smem_raw) & 1023) __trap();
  }
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::kTileBytes;
  uint8_t* sStage = sV + C::kTileBytes;  // ST x {Q, dO, lse[128], D[128]}
  uint8_t* sdS = sStage + ST * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + C::kDsBytes);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = qdo_full + ST;
  uint64_t* s_full = qdo_empty + ST;
  uint64_t* p_full = s_full + 1;
  uint64_t* dp_full = p_full + 1;
  uint64_t* ds_full = dp_full + 1;
  uint64_t* sds_empty = ds_full + 1;
  uint64_t* dq_full = sds_empty + 1;
  uint64_t* dq_empty = dq_full + 1;
  uint64_t* acc_full = dq_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int kt = blockIdx.x, head = blockIdx.y, bi = blockIdx.z;
  const int kv_row0 = bi * P.s + kt * kTile;
  const int q_row_base = bi * P.s;
  const int col0 = head * HD;
  const long long stat0 = ((long long)bi * P.h + head) * P.s;
  long long* const tr = (kt == 0 && head == 0 && bi == 0) ? P.trace : nullptr;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  auto sQ = [&](int st) { return sStage + st * C::kStageBytes; };
  auto sdO = [&](int st) { return sStage + st * C::kStageBytes + C::kTileBytes; };
  auto sLse = [&](int st) { return reinterpret_cast<float*>(sStage + st * C::kStageBytes + 2 * C::kTileBytes); };
  auto sD = [&](int st) { return sLse(st) + kTile; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
    tma_prefetch_desc(&P.tdo);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(kv_full, 1);
      for (int s = 0; s < ST; ++s) {
        mbar_init(&qdo_full[s], 1);
        mbar_init(&qdo_empty[s], 1);
      }
      mbar_init(s_full, 1);
      mbar_init(p_full, 8);
      mbar_init(dp_full, 1);
      mbar_init(ds_full, 8);
      mbar_init(sds_empty, 1);
      mbar_init(dq_full, 1);
      mbar_init(dq_empty, 4);
      mbar_init(acc_full, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(kv_full, 2 * C::kTileBytes);
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_2d(sK + c * kTile * 128, &P.tk, kv_full, col0 + 64 * c, kv_row0);
        tma_load_2d(sV + c * kTile * 128, &P.tv, kv_full, col0 + 64 * c, kv_row0);
      }
      for (int i = 0; i < P.n_q; ++i) {
        const int st = i % ST;
        const uint32_t ph = (i / ST) & 1;
        mbar_wait(&qdo_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], C::kStageBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(sQ(st) + c * kTile * 128, &P.tq, &qdo_full[st], col0 + 64 * c, q_row_base + i * kTile);
          tma_load_2d(sdO(st) + c * kTile * 128, &P.tdo, &qdo_full[st], col0 + 64 * c, q_row_base + i * kTile);
        }
        bulk_load_1d(sLse(st), P.lse + stat0 + i * kTile, kTile * 4, &qdo_full[st]);
        bulk_load_1d(sD(st), P.D + stat0 + i * kTile, kTile * 4, &qdo_full[st]);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_ss = make_idesc_bf16_f32(kTile, kTile, false, false);  // [1], [2]
    constexpr uint32_t idesc_ts = make_idesc_bf16_f32(kTile, HD, false, true);      // [3], [4]
    constexpr uint32_t idesc_dq = make_idesc_bf16_f32(kTile, HD, true, true);       // [5]
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV), ds_base = smem_u32(sdS);
    auto mma_ss = [&](uint32_t d, uint32_t a_base, uint32_t b_base) {  // K-major x K-major over hd
#pragma unroll
      for (int k = 0; k < HD / 16; ++k) {
        const uint32_t off = (k >> 2) * kTile * 128 + (k & 3) * 32;
        umma_bf16(d, make_sw128_desc(a_base + off, 16, 1024), make_sw128_desc(b_base + off, 16, 1024), idesc_ss,
                  k > 0 ? 1u : 0u);
      }
    };
    // over 128 query rows; A = P^T / dS^T bf16 pairs: queries [64g, 64g + 64) at TMEM columns [64g, 64g + 32)
    auto mma_ts = [&](uint32_t d, uint32_t a_tmem, uint32_t b_base, bool acc) {
#pragma unroll
      for (int k = 0; k < kTile / 16; ++k)
        umma_bf16_ts(d, a_tmem + (k >> 2) * 64 + (k & 3) * 8, make_sw128_desc(b_base + k * 2048, kTile * 128, 1024),
                     idesc_ts,
                     (acc || k > 0) ? 1u : 0u);
    };
    mbar_wait(kv_full, 0);
    mbar_wait(&qdo_full[0], 0);
    tc_fence_after();
    if (elect_one()) {
      mma_ss(tmem + C::tS, k_base, smem_u32(sQ(0)));
      umma_commit(s_full);
      mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(0)));
      umma_commit(dp_full);
    }
    __syncwarp();
    for (int i = 0; i < P.n_q; ++i) {
      const int st = i % ST;
      const uint32_t ph = i & 1;
      mbar_wait(p_full, ph);
      BTP_STAMP(8);
      tc_fence_after();
      if (elect_one()) mma_ts(tmem + C::tdV, tmem + C::tS, smem_u32(sdO(st)), i > 0);  // [3]
      __syncwarp();
      const bool more = i + 1 < P.n_q;
      const int st1 = (i + 1) % ST;
      if (more) {
        mbar_wait(&qdo_full[st1], ((i + 1) / ST) & 1);
        tc_fence_after();
        if (elect_one()) {
          mma_ss(tmem + C::tS, k_base, smem_u32(sQ(st1)));  // [1]_{i+1}
          umma_commit(s_full);
        }
        __syncwarp();
      }
      BTP_STAMP(9);
      mbar_wait(ds_full, ph);
      BTP_STAMP(10);
      tc_fence_after();
      if (elect_one()) {
        mma_ts(tmem + C::tdK, tmem + C::tdP, smem_u32(sQ(st)), i > 0);  // [4]
        umma_commit(&qdo_empty[st]);
      }
      __syncwarp();
      if (i > 0) {
        mbar_wait(dq_empty, (i - 1) & 1);
        tc_fence_after();
      }
      BTP_STAMP(11);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)  // [5]: A = dS (MN-major, 2 chunks of 64 queries), B = K (MN-major)
          umma_bf16(tmem + C::tdQ, make_sw128_desc(ds_base + k * 2048, kTile * 128, 1024),
                    make_sw128_desc(k_base + k * 2048, kTile * 128, 1024), idesc_dq, k > 0 ? 1u : 0u);
        umma_commit(dq_full);
        umma_commit(sds_empty);
      }
      __syncwarp();
      if (more) {
        if constexpr (C::tdQ == C::tdP) {
          mbar_wait(dq_empty, i & 1);  // dQ_i must be drained before dP^T_{i+1} overwrites it
          tc_fence_after();
        }
        if (elect_one()) {
          mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(st1)));  // [2]_{i+1}
          umma_commit(dp_full);
        }
        __syncwarp();
        BTP_STAMP(12);
      }
    }
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
  } else if (warp < 10) {
    // ---------------------------------------------------------------- compute warps 2..9
    // Two warps per TMEM lane quarter: group g handles query columns [64g, 64g + 64) of the tile and
    // writes its bf16 P^T / dS^T pairs over TMEM columns [64g, 64g + 32) of the S / dP blocks, which
    // only it reads (the MMA A-operand addresses follow that split).
    const uint32_t g = (warp - 2) >> 2;
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // key row within the tile == TMEM lane
    const uint32_t lane_addr = (q4 * 32) << 16;
    const float2 c2 = make_float2(P.c, P.c);
    const uint32_t ds_row = smem_u32(sdS) + g * (kTile * 128) + row * 128;
    for (int i = 0; i < P.n_q; ++i) {
      const int st = i % ST;
      const uint32_t ph = i & 1;
      const uint32_t lse_a = smem_u32(sLse(st)) + g * 256, d_a = smem_u32(sD(st)) + g * 256;
      mbar_wait(&qdo_full[st], (i / ST) & 1);  // lse / D of this query tile are resident
      mbar_wait(s_full, ph);
      if (q4 == 2) BTP_STAMP(4 * g);
      tc_fence_after();
      // P^T kept as packed bf16 pairs (the values the dV MMA consumes) for dS below
      uint32_t pk[32];
      {
        float sv[64];
        tmem_ld_32x32b_x64(tmem + C::tS + lane_addr + g * 64, *reinterpret_cast<uint32_t(*)[64]>(&sv[0]));
        tmem_ld_wait();
#pragma unroll
        for (int m = 0; m < 64; m += 4) {
          const float4 l4 = ld_shared_f4(lse_a + m * 4);
          const float2 x01 = ffma2(make_float2(sv[m], sv[m + 1]), c2, make_float2(-l4.x, -l4.y));
          const float2 x23 = ffma2(make_float2(sv[m + 2], sv[m + 3]), c2, make_float2(-l4.z, -l4.w));
          pk[m / 2] = pack_bf16(ex2_approx(x01.x), ex2_approx(x01.y));
          pk[m / 2 + 1] = pack_bf16(ex2_approx(x23.x), ex2_approx(x23.y));
        }
      }
      tmem_st_32x32b_x32(tmem + C::tS + lane_addr + g * 64, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (q4 == 2) BTP_STAMP(4 * g + 1);
      // dS^T = P^T (dP^T - D)
      mbar_wait(dp_full, ph);
      tc_fence_after();
      if (i > 0) mbar_wait(sds_empty, (i - 1) & 1);  // dQ_{i-1} has read the previous dS
      if (q4 == 2) BTP_STAMP(4 * g + 2);
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {  // 32 query columns per step
        uint32_t dp[32];
        tmem_ld_32x32b_x32(tmem + C::tdP + lane_addr + g * 64 + cc * 32, dp);
        tmem_ld_wait();
        uint32_t ds[16];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 d4 = ld_shared_f4(d_a + (cc * 32 + j) * 4);
          const uint32_t p01 = pk[(cc * 32 + j) / 2], p23 = pk[(cc * 32 + j) / 2 + 1];
          const float2 a01 = fmul2(make_float2(bf16_lo(p01), bf16_hi(p01)),
                                   fadd2(make_float2(__uint_as_float(dp[j]), __uint_as_float(dp[j + 1])),
                                         make_float2(-d4.x, -d4.y)));
          const float2 a23 = fmul2(make_float2(bf16_lo(p23), bf16_hi(p23)),
                                   fadd2(make_float2(__uint_as_float(dp[j + 2]), __uint_as_float(dp[j + 3])),
                                         make_float2(-d4.z, -d4.w)));
          ds[j / 2] = pack_bf16(a01.x, a01.y);
          ds[j / 2 + 1] = pack_bf16(a23.x, a23.y);
        }
        // TMEM columns [64g + 16cc, +16) of the dP block (already read) take dS^T
        tmem_st_32x32b_x16(tmem + C::tdP + lane_addr + g * 64 + cc * 16, ds);
        // shared: chunk g (64 queries), row = key, 16-byte units 4cc .. 4cc + 3, 128B swizzle
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t unit = cc * 4 + u;
          st_shared_v4(ds_row + ((unit ^ (row & 7)) << 4), ds[4 * u], ds[4 * u + 1], ds[4 * u + 2], ds[4 * u + 3]);
        }
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (q4 == 2) BTP_STAMP(4 * g + 3);
    }
    // ---------------------------------------------------------------- dK / dV epilogue (group 0: dV, 1: dK)
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t tcol = g == 0 ? C::tdV : C::tdK;
    const float sc = g == 0 ? 1.f : P.dk_scale;
    __nv_bfloat16* out = g == 0 ? P.dv + (long long)(kv_row0 + row) * P.lddv + col0
                                : P.dk + (long long)(kv_row0 + row) * P.lddk + col0;
#pragma unroll
    for (int cc = 0; cc < HD / 32; ++cc) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tmem + tcol + lane_addr + cc * 32, o);
      tmem_ld_wait();
      uint32_t ok[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) ok[j] = pack_bf16(__uint_as_float(o[2 * j]) * sc, __uint_as_float(o[2 * j + 1]) * sc);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_global_v4(out + cc * 32 + v * 8, make_uint4(ok[4 * v], ok[4 * v + 1], ok[4 * v + 2], ok[4 * v + 3]));
    }
  } else {
    // ---------------------------------------------------------------- dQ reduce warps 10..13
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // query row within the tile
    const uint32_t lane_addr = (q4 * 32) << 16;
    for (int i = 0; i < P.n_q; ++i) {
      mbar_wait(dq_full, i & 1);
      if (q4 == 2) BTP_STAMP(13);
      tc_fence_after();
      float* dst = P.dq_acc + (long long)(q_row_base + i * kTile + row) * P.ldacc + col0;
#pragma unroll
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + C::tdQ + lane_addr + cc * 32, o);
        tmem_ld_wait();
        if (cc == HD / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_empty);  // TMEM drained; the adds below only touch registers
        }
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          red_add_v4(dst + cc * 32 + j, __uint_as_float(o[j]), __uint_as_float(o[j + 1]), __uint_as_float(o[j + 2]),
                     __uint_as_float(o[j + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------- backward, hd 64
// At hd = 64 the three N = hd products (dV, dK, dQ) run at half the tensor rate (an M128 x N64 x K16
// tcgen05.mma costs the same ~64 cycles as N128: scripts/microbench/mma_rates.cu), so the tensor pipe
// is the bound and must never wait. Differences from the generic kernel above:
//   * dS^T is NOT written back to TMEM: the dK MMA reads it from the same shared-memory tile the dQ
//     MMA uses (rows = key, 128 B of queries per row: K-major for A = dS^T, MN-major for A = dS);
//   * so the dP^T block is free as soon as the compute warps hold dP^T in registers (dp_read), and
//     dP^T of the next query tile is issued BEFORE this tile's dK / dQ MMAs;
//   * dS (shared) and dQ (TMEM, columns 384 / 448) are double-buffered, so neither the compute warps
//     nor the MMA issuer wait on the previous tile's dQ MMA or its reduction.
// Tensor order per tile:  [3]_i dV  [1]_{i+1} S^T  [2]_{i+1} dP^T  [4]_i dK  [5]_i dQ.
struct Bwd64Cfg {
  static constexpr int HD = 64;
  static constexpr int ST = 3;                                       // Q / dO / lse / D ring
  static constexpr int kTileBytes = kTile * HD * 2;                 // 16 KB
  static constexpr int kStageBytes = 2 * kTileBytes + 2 * kTile * 4;  // Q, dO, lse, D
  static constexpr int kDsBytes = kTile * kTile * 2;                  // 32 KB per buffer
  static constexpr int kBarBytes = 256;
  static constexpr int kDqBytes = kTile * 32 * 4;                    // fp32 dQ staging: one 32-column box
  static constexpr int kSmem = 1024 + 2 * kTileBytes + ST * kStageBytes + 2 * kDsBytes + kDqBytes + kBarBytes;
  static constexpr int kThreads = 448;
  static constexpr uint32_t tS = 0, tdP = 128, tdV = 256, tdK = 320, tdQ = 384;  // dQ: 384 / 448
};

// kPk (btp_attn_tune(3, 2)): the dS phase computes P^T (dP^T - D) from the bf16 P^T pairs the P phase
// already packed for the dV MMA (32 registers instead of 64 fp32), so the whole 64-column dP^T block
// fits in registers at once: ONE x64 TMEM load, and dp_read (which gates the next tile's dP^T MMA)
// arrives before any dS math instead of after the first 32-column half.
template <bool kTrace, int kPoly, bool kPk = false>
__global__ void __launch_bounds__(448, 1) attn_bwd64_kernel(const __grid_constant__ BwdParams P) {
  using C = Bwd64Cfg;
  constexpr int HD = 64, ST = C::ST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::kTileBytes;
  uint8_t* sStage = sV + C::kTileBytes;
  uint8_t* sdS = sStage + ST * C::kStageBytes;  // 2 buffers
  float* sdQ = reinterpret_cast<float*>(sdS + 2 * C::kDsBytes);  // fp32 [128][32] staging (one box at a time)
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sdQ) + C::kDqBytes);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;        // [ST]
  uint64_t* qdo_empty = qdo_full + ST;  // [ST]
  uint64_t* s_full = qdo_empty + ST;
  uint64_t* p_full = s_full + 1;
  uint64_t* dp_full = p_full + 1;
  uint64_t* dp_read = dp_full + 1;
  uint64_t* ds_full = dp_read + 1;
  uint64_t* sds_empty = ds_full + 1;   // [2]
  uint64_t* dq_full = sds_empty + 2;   // [2]
  uint64_t* dq_empty = dq_full + 2;    // [2]
  uint64_t* acc_full = dq_empty + 2;
  uint64_t* acc_empty = acc_full + 1;  // persistent: the compute warps have read this item's dK / dV
  uint64_t* kv_empty = acc_empty + 1;  // persistent: the item's last MMA reading K / V is done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + 1);

  // Work items (key tile kt of head `head` of sequence bi) are walked persistently: CTA x takes items
  // x, x + gridDim.x, ... (with gridDim.x == n_items every CTA has one). Per-tile barrier phases, the
  // Q / dO ring and the dS / dQ double buffers run on the CTA's global tile counter g = it * n_q + i,
  // so the next item's loads and first MMAs overlap this item's dQ-reduce tail and dK / dV stores.
  struct Item {
    int kv_row0, q_row_base, col0;
    long long stat0;
  };
  auto item_of = [&](int it) {
    const int item = (int)blockIdx.x + it * (int)gridDim.x;
    const int kt = item % P.n_q, r = item / P.n_q;
    const int head = r % P.h, bi = r / P.h;
    return Item{bi * P.s + kt * kTile, bi * P.s, head * HD, ((long long)bi * P.h + head) * P.s};
  };
  const int n_it = ((int)blockIdx.x < P.n_items) ? (P.n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // kTrace: every CTA's (SM id, start, walk done, end) clock64 stamps after the per-tile stamps
  long long* const ct =
      kTrace ? P.trace + (long long)P.n_q * 16 + 8ll * blockIdx.x : nullptr;
  if (kTrace && threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    ct[0] = sm;
    ct[1] = clock64();
  }
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  auto sQ = [&](int st) { return sStage + st * C::kStageBytes; };
  auto sdO = [&](int st) { return sStage + st * C::kStageBytes + C::kTileBytes; };
  auto sLse = [&](int st) { return reinterpret_cast<float*>(sStage + st * C::kStageBytes + 2 * C::kTileBytes); };
  auto sD = [&](int st) { return sLse(st) + kTile; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
    tma_prefetch_desc(&P.tdo);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(kv_full, 1);
      for (int s = 0; s < ST; ++s) {
        mbar_init(&qdo_full[s], 1);
        mbar_init(&qdo_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&sds_empty[s], 1);
        mbar_init(&dq_full[s], 1);
        mbar_init(&dq_empty[s], 4);
      }
      mbar_init(s_full, 1);
      mbar_init(p_full, 8);
      mbar_init(dp_full, 1);
      mbar_init(dp_read, 8);
      mbar_init(ds_full, 8);
      mbar_init(acc_full, 1);
      mbar_init(acc_empty, 8);
      mbar_init(kv_empty, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      for (int it = 0; it < n_it; ++it) {
        const Item w = item_of(it);
        // K / V of item `it` once the previous item's last MMA has read them; issued after the first
        // ring tiles of this item (whose slots free up earlier) so those loads are not held back
        auto load_kv = [&]() {
          if (it > 0) mbar_wait(kv_empty, (it - 1) & 1);
          mbar_arrive_expect_tx(kv_full, 2 * C::kTileBytes);
          tma_load_2d(sK, &P.tk, kv_full, w.col0, w.kv_row0);
          tma_load_2d(sV, &P.tv, kv_full, w.col0, w.kv_row0);
        };
        const int kv_at = P.n_q < ST ? P.n_q : ST;
        for (int i = 0; i < P.n_q; ++i) {
          if (i == kv_at) load_kv();
          const int g = it * P.n_q + i;
          const int st = g % ST;
          mbar_wait(&qdo_empty[st], ((g / ST) & 1) ^ 1);
          mbar_arrive_expect_tx(&qdo_full[st], C::kStageBytes);
          tma_load_2d(sQ(st), &P.tq, &qdo_full[st], w.col0, w.q_row_base + i * kTile);
          tma_load_2d(sdO(st), &P.tdo, &qdo_full[st], w.col0, w.q_row_base + i * kTile);
          bulk_load_1d(sLse(st), P.lse + w.stat0 + i * kTile, kTile * 4, &qdo_full[st]);
          bulk_load_1d(sD(st), P.D + w.stat0 + i * kTile, kTile * 4, &qdo_full[st]);
        }
        if (kv_at == P.n_q) load_kv();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_ss = make_idesc_bf16_f32(kTile, kTile, false, false);  // [1], [2]
    constexpr uint32_t idesc_ts = make_idesc_bf16_f32(kTile, HD, false, true);      // [3], [4]
    constexpr uint32_t idesc_dq = make_idesc_bf16_f32(kTile, HD, true, true);       // [5]
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
    auto mma_ss = [&](uint32_t d, uint32_t a_base, uint32_t b_base) {  // K-major x K-major over hd = 64
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_bf16(d, make_sw128_desc(a_base + k * 32, 16, 1024), make_sw128_desc(b_base + k * 32, 16, 1024), idesc_ss,
                  k > 0 ? 1u : 0u);
    };
    for (int it = 0; it < n_it; ++it) {
    long long* const tr = (kTrace && blockIdx.x == 0 && it == 0) ? P.trace : nullptr;
    const int g0 = it * P.n_q;
    mbar_wait(kv_full, it & 1);
    mbar_wait(&qdo_full[g0 % ST], (g0 / ST) & 1);
    if (it > 0) mbar_wait(dp_read, (g0 - 1) & 1);  // the previous item's last dP^T is in registers
    tc_fence_after();
    if (elect_one()) {
      mma_ss(tmem + C::tS, k_base, smem_u32(sQ(g0 % ST)));
      umma_commit(s_full);
      mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(g0 % ST)));
      umma_commit(dp_full);
    }
    __syncwarp();
    for (int i = 0; i < P.n_q; ++i) {
      const int g = g0 + i;
      const int st = g % ST, buf = g & 1;  // Q/dO ring stage; dS / dQ double-buffer parity
      const uint32_t ph = g & 1;
      const bool more = i + 1 < P.n_q;
      const int st1 = (g + 1) % ST;
      mbar_wait(p_full, ph);
      if (i == 0 && it > 0) mbar_wait(acc_empty, (it - 1) & 1);  // dV / dK of the previous item are read
      BTP_STAMP64(8);
      tc_fence_after();
      if (elect_one()) {  // [3] dV += P^T dO: A = P^T pairs, queries [64g, +64) at TMEM columns [64g, +32)
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + C::tdV, tmem + C::tS + (k >> 2) * 64 + (k & 3) * 8,
                       make_sw128_desc(smem_u32(sdO(st)) + k * 2048, kTile * 128, 1024), idesc_ts,
                       (i > 0 || k > 0) ? 1u : 0u);
      }
      __syncwarp();
      if (more) {
        mbar_wait(&qdo_full[st1], ((g + 1) / ST) & 1);
        tc_fence_after();
        if (elect_one()) {
          mma_ss(tmem + C::tS, k_base, smem_u32(sQ(st1)));  // [1]_{i+1}
          umma_commit(s_full);
        }
        __syncwarp();
        mbar_wait(dp_read, ph);  // the compute warps hold dP^T_i in registers
        tc_fence_after();
        if (elect_one()) {
          mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(st1)));  // [2]_{i+1}
          umma_commit(dp_full);
        }
        __syncwarp();
      }
      BTP_STAMP64(9);
      mbar_wait(ds_full, ph);
      BTP_STAMP64(10);
      tc_fence_after();
      const uint32_t ds_base = smem_u32(sdS + buf * C::kDsBytes);
      if (elect_one()) {
        // [4] dK += dS^T Q: A = dS^T K-major in shared memory (chunk g = queries [64g, +64), 128 B rows)
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16(tmem + C::tdK, make_sw128_desc(ds_base + (k >> 2) * (kTile * 128) + (k & 3) * 32, 16, 1024),
                    make_sw128_desc(smem_u32(sQ(st)) + k * 2048, kTile * 128, 1024), idesc_ts,
                    (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&qdo_empty[st]);
      }
      __syncwarp();
      if (g >= 2) {
        mbar_wait(&dq_empty[buf], ((g >> 1) - 1) & 1);
        tc_fence_after();
      }
      BTP_STAMP64(11);
      if (elect_one()) {
        // [5] dQ_i = dS K: A = dS MN-major (the same tile), B = K MN-major
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16(tmem + C::tdQ + buf * 64, make_sw128_desc(ds_base + k * 2048, kTile * 128, 1024),
                    make_sw128_desc(k_base + k * 2048, kTile * 128, 1024), idesc_dq, k > 0 ? 1u : 0u);
        umma_commit(&dq_full[buf]);
        umma_commit(&sds_empty[buf]);
        if (!more) umma_commit(kv_empty);  // the item's last MMA on K / V
      }
      __syncwarp();
      BTP_STAMP64(12);
    }
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
    if (kTrace && lane == 0) ct[2] = clock64();  // last MMA issued
    }
  } else if (warp < 10) {
    // ---------------------------------------------------------------- compute warps 2..9
    const uint32_t g = (warp - 2) >> 2;
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // key row within the tile == TMEM lane
    const uint32_t lane_addr = (q4 * 32) << 16;
    const float2 c2 = make_float2(P.c, P.c);
    for (int it = 0; it < n_it; ++it) {
    long long* const tr = (kTrace && blockIdx.x == 0 && it == 0) ? P.trace : nullptr;
    const Item w = item_of(it);
    for (int i = 0; i < P.n_q; ++i) {
      const int gt = it * P.n_q + i;
      const int st = gt % ST, buf = gt & 1;
      const uint32_t ph = gt & 1;
      const uint32_t lse_a = smem_u32(sLse(st)) + g * 256, d_a = smem_u32(sD(st)) + g * 256;
      mbar_wait(&qdo_full[st], (gt / ST) & 1);  // lse / D of this query tile are resident
      mbar_wait(s_full, ph);
      if (q4 == 2) BTP_STAMP64(4 * g);
      tc_fence_after();
      // P^T in fp32 registers for dS below; its bf16 pairs go to TMEM for the dV MMA
      float pv[64];
      uint32_t pk[32];
      tmem_ld_32x32b_x64(tmem + C::tS + lane_addr + g * 64, *reinterpret_cast<uint32_t(*)[64]>(&pv[0]));
      tmem_ld_wait();
      if (q4 == 2 && g == 0) BTP_STAMP64(14);
      {
#pragma unroll
        for (int m = 0; m < 64; m += 4) {
          const float4 l4 = ld_shared_f4(lse_a + m * 4);
          const float2 x01 = ffma2(make_float2(pv[m], pv[m + 1]), c2, make_float2(-l4.x, -l4.y));
          const float2 x23 = ffma2(make_float2(pv[m + 2], pv[m + 3]), c2, make_float2(-l4.z, -l4.w));
          float2 e01, e23;
          e01.x = ex2_approx(x01.x);
          e01.y = ex2_approx(x01.y);
          if (kPoly > 0 && ((m / 4) % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
            e23 = ex2_poly2(x23);  // a share of the exp2s on the FMA pipe (the MUFU bounds this phase)
          } else {
            e23.x = ex2_approx(x23.x);
            e23.y = ex2_approx(x23.y);
          }
          pv[m] = e01.x;
          pv[m + 1] = e01.y;
          pv[m + 2] = e23.x;
          pv[m + 3] = e23.y;
          pk[m / 2] = pack_bf16(e01.x, e01.y);
          pk[m / 2 + 1] = pack_bf16(e23.x, e23.y);
        }
        if (q4 == 2 && g == 0) BTP_STAMP64(15);
        tmem_st_32x32b_x32(tmem + C::tS + lane_addr + g * 64, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (q4 == 2) BTP_STAMP64(4 * g + 1);
      mbar_wait(dp_full, ph);
      tc_fence_after();
      if (gt >= 2) mbar_wait(&sds_empty[buf], ((gt >> 1) - 1) & 1);  // dQ_{i-2} has read this dS buffer
      if (q4 == 2) BTP_STAMP64(4 * g + 2);
      const uint32_t ds_row = smem_u32(sdS + buf * C::kDsBytes) + g * (kTile * 128) + row * 128;
      if constexpr (kPk) {
        uint32_t dp[64];
        tmem_ld_32x32b_x64(tmem + C::tdP + lane_addr + g * 64, dp);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_read);  // the next tile's dP^T MMA may overwrite the block now
#pragma unroll
        for (int unit = 0; unit < 8; ++unit) {  // 8 queries per 16-byte unit
          uint32_t ds[4];
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            const int m = unit * 8 + j;
            const float4 d4 = ld_shared_f4(d_a + m * 4);
            const float2 p01 = make_float2(__uint_as_float(pk[m / 2] << 16), __uint_as_float(pk[m / 2] & 0xffff0000u));
            const float2 p23 =
                make_float2(__uint_as_float(pk[m / 2 + 1] << 16), __uint_as_float(pk[m / 2 + 1] & 0xffff0000u));
            const float2 a01 = fmul2(p01, fadd2(make_float2(__uint_as_float(dp[m]), __uint_as_float(dp[m + 1])),
                                                make_float2(-d4.x, -d4.y)));
            const float2 a23 = fmul2(p23, fadd2(make_float2(__uint_as_float(dp[m + 2]), __uint_as_float(dp[m + 3])),
                                                make_float2(-d4.z, -d4.w)));
            ds[j / 2] = pack_bf16(a01.x, a01.y);
            ds[j / 2 + 1] = pack_bf16(a23.x, a23.y);
          }
          st_shared_v4(ds_row + ((unit ^ (row & 7)) << 4), ds[0], ds[1], ds[2], ds[3]);
        }
      } else {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // 32 queries per half
        uint32_t dp[32];
        tmem_ld_32x32b_x32(tmem + C::tdP + lane_addr + g * 64 + hh * 32, dp);
        tmem_ld_wait();
        if (hh == 1) {  // dP^T of this tile is in registers: the next tile's dP^T MMA may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_read);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // 8 queries per 16-byte unit
          uint32_t ds[4];
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            const int mm = u * 8 + j, m = hh * 32 + mm;
            const float4 d4 = ld_shared_f4(d_a + m * 4);
            const float2 a01 = fmul2(make_float2(pv[m], pv[m + 1]),
                                     fadd2(make_float2(__uint_as_float(dp[mm]), __uint_as_float(dp[mm + 1])),
                                           make_float2(-d4.x, -d4.y)));
            const float2 a23 = fmul2(make_float2(pv[m + 2], pv[m + 3]),
                                     fadd2(make_float2(__uint_as_float(dp[mm + 2]), __uint_as_float(dp[mm + 3])),
                                           make_float2(-d4.z, -d4.w)));
            ds[j / 2] = pack_bf16(a01.x, a01.y);
            ds[j / 2 + 1] = pack_bf16(a23.x, a23.y);
          }
          const uint32_t unit = hh * 4 + u;
          st_shared_v4(ds_row + ((unit ^ (row & 7)) << 4), ds[0], ds[1], ds[2], ds[3]);
        }
      }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (q4 == 2) BTP_STAMP64(4 * g + 3);
    }
    // ---------------------------------------------------------------- dK / dV epilogue (group 0: dV, 1: dK)
    if (kTrace && warp == 2 && lane == 0) ct[3] = clock64();  // compute walk done
    mbar_wait(acc_full, it & 1);
    tc_fence_after();
    const uint32_t tcol = g == 0 ? C::tdV : C::tdK;
    const float sc = g == 0 ? 1.f : P.dk_scale;
    __nv_bfloat16* out = g == 0 ? P.dv + (long long)(w.kv_row0 + row) * P.lddv + w.col0
                                : P.dk + (long long)(w.kv_row0 + row) * P.lddk + w.col0;
    uint32_t o[64];
    tmem_ld_32x32b_x64(tmem + tcol + lane_addr, o);
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_empty);  // the next item's first dV / dK MMA may overwrite them
#pragma unroll
    for (int cc = 0; cc < HD / 32; ++cc) {
      uint32_t ok[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        ok[j] = pack_bf16(__uint_as_float(o[cc * 32 + 2 * j]) * sc, __uint_as_float(o[cc * 32 + 2 * j + 1]) * sc);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_global_v4(out + cc * 32 + v * 8, make_uint4(ok[4 * v], ok[4 * v + 1], ok[4 * v + 2], ok[4 * v + 3]));
    }
    if (kTrace && warp == 2 && lane == 0) ct[7] = clock64();  // dK / dV stored
    }
  } else {
    // ---------------------------------------------------------------- dQ reduce warps 10..13
    // TMEM -> registers -> 128B-swizzled fp32 smem tile -> TMA reduce-add into the fp32 accumulator
    // (the add happens in L2; no per-thread red.global traffic in the LSU queue the compute warps use)
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // query row within the tile
    const uint32_t lane_addr = (q4 * 32) << 16;
    const bool issuer = (warp == 10 && lane == 0);
    for (int it = 0; it < n_it; ++it) {
    long long* const tr = (kTrace && blockIdx.x == 0 && it == 0) ? P.trace : nullptr;
    const Item w = item_of(it);
    for (int i = 0; i < P.n_q; ++i) {
      const int gt = it * P.n_q + i;
      const int buf = gt & 1;
      mbar_wait(&dq_full[buf], (gt >> 1) & 1);
      if (q4 == 2) BTP_STAMP64(13);
      tc_fence_after();
      uint32_t o[64];
      tmem_ld_32x32b_x64(tmem + C::tdQ + buf * 64 + lane_addr, o);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_empty[buf]);
#pragma unroll
      for (int bx = 0; bx < 2; ++bx) {  // one 32-column box at a time through the 16 KB staging tile
        if (issuer) bulk_wait_read<0>();  // the previous box's reduce has read the staging tile
        named_bar_sync(1, 128);
        const uint32_t base = smem_u32(sdQ) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(base + ((u ^ (row & 7)) << 4), o[bx * 32 + 4 * u], o[bx * 32 + 4 * u + 1],
                       o[bx * 32 + 4 * u + 2], o[bx * 32 + 4 * u + 3]);
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (issuer) {
          tma_reduce_add_2d(&P.tdq, sdQ, w.col0 + 32 * bx, w.q_row_base + i * kTile);
          bulk_commit();
        }
      }
    }
    }
    if (kTrace && issuer) ct[4] = clock64();
    if (issuer) bulk_wait<0>();
    if (kTrace && issuer) ct[5] = clock64();
    __syncwarp();  // the issuer lane rejoins its warp before the final barrier (bar.sync is per warp)
  }
  tc_fence_before();
  __syncthreads();
  if (kTrace && threadIdx.x == 0) ct[6] = clock64();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------- backward, hd 64, split roles
// The kernel above runs the P phase (MUFU-bound: exp2) and the dS phase (FMA / ALU: P (dP - D), pack,
// store) on the SAME 8 warps, one after the other, so each pipe idles half the time and the loop is
// ~3100 cycles per query tile against a ~2160-cycle tensor floor (profiles/attention). Here the roles
// are split so P of tile i+1 overlaps dS of tile i:
//   w2..w9   P warps (two per scheduler, 64 query columns each): S^T -> P^T = exp2(S^T c - lse) ->
//            bf16 pairs into their own TMEM block (tP), read by the dV MMA and by the dS warps
//   w10..w17 dS warps, two groups of four alternating query tiles (group = tile parity; one warp per
//            scheduler per group, a key row's 128 queries each, in 32-column chunks): dP^T and P^T from
//            TMEM -> dS^T = P^T (dP^T - D) -> bf16, swizzled into shared memory (the A operand of the dK
//            MMA, K-major, and of the dQ MMA, MN-major). The stores must be made visible to the tensor
//            core (fence.proxy.async per writing thread), which under the MMAs' shared-memory traffic
//            costs ~1000 cycles per tile (measured: 1.85 ms with vs 1.28 ms without); alternating groups
//            give each group two tile periods, so one group's fence drains while the other computes.
//            Barriers between the dS groups and the other roles are per tile parity.
//   w18..w21 dQ reduce warps (TMEM -> swizzled fp32 smem tile -> TMA reduce-add)
// TMEM: S^T 0..127, P^T 128..191, dP^T 192..319, dV 320..383, dK 384..447, dQ 448..511.
// Tensor order per tile: [1]_{i+1} S^T  [3]_i dV  [2]_{i+1} dP^T  [4]_i dK  [5]_i dQ.
struct Bwd64sCfg {
  static constexpr int HD = 64;
  static constexpr int kTileBytes = kTile * HD * 2;                   // 16 KB
  static constexpr int kStageBytes = 2 * kTileBytes + 2 * kTile * 4;  // Q, dO, lse, D
  static constexpr int kDsBytes = kTile * kTile * 2;                  // 32 KB per buffer
  static constexpr int ST = 3;                                        // Q / dO / lse / D ring
  static constexpr int kDqBytes = kTile * 32 * 4;                     // one 32-column fp32 box of dQ
  static constexpr int kBarBytes = 256;
  static constexpr int kSmem = 1024 + 2 * kTileBytes + ST * kStageBytes + 2 * kDsBytes + kDqBytes + kBarBytes;
  static constexpr int kThreads = 704;
  static constexpr uint32_t tS = 0, tP = 128, tdP = 192, tdV = 320, tdK = 384, tdQ = 448;
};

__global__ void __launch_bounds__(704, 1) attn_bwd64s_kernel(const __grid_constant__ BwdParams P) {
  using C = Bwd64sCfg;
  constexpr int HD = 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::kTileBytes;
  uint8_t* sStage = sV + C::kTileBytes;
  uint8_t* sdS = sStage + C::ST * C::kStageBytes;  // 2 buffers
  float* sdQ = reinterpret_cast<float*>(sdS + 2 * C::kDsBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sdQ) + C::kDqBytes);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;           // [ST]
  uint64_t* qdo_empty = qdo_full + C::ST;  // [ST]
  uint64_t* sds_empty = qdo_empty + C::ST; // [2]
  uint64_t* s_full = sds_empty + 2;
  uint64_t* s_read = s_full + 1;
  uint64_t* p_full = s_read + 1;    // [2] by tile parity
  uint64_t* p_empty = p_full + 2;   // [2]
  uint64_t* dp_full = p_empty + 2;  // [2]
  uint64_t* dp_read = dp_full + 2;  // [2]
  uint64_t* ds_full = dp_read + 2;  // [2]
  uint64_t* dq_full = ds_full + 2;
  uint64_t* dq_empty = dq_full + 1;
  uint64_t* acc_full = dq_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int kt = blockIdx.x, head = blockIdx.y, bi = blockIdx.z;
  const int kv_row0 = bi * P.s + kt * kTile;
  const int q_row_base = bi * P.s;
  const int col0 = head * HD;
  const long long stat0 = ((long long)bi * P.h + head) * P.s;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  long long* const tr = (kt == 0 && head == 0 && bi == 0) ? P.trace : nullptr;
#define SSTAMP(e)                                                   \
  do {                                                              \
    if (tr != nullptr && lane == 0) tr[i * 16 + (e)] = clock64();   \
  } while (0)
  auto sQ = [&](int st) { return sStage + st * C::kStageBytes; };
  auto sdO = [&](int st) { return sStage + st * C::kStageBytes + C::kTileBytes; };
  auto sLse = [&](int st) { return reinterpret_cast<float*>(sStage + st * C::kStageBytes + 2 * C::kTileBytes); };
  auto sD = [&](int st) { return sLse(st) + kTile; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&P.tq);
    tma_prefetch_desc(&P.tk);
    tma_prefetch_desc(&P.tv);
    tma_prefetch_desc(&P.tdo);
  }
  if (warp == 1) {
    if (lane == 0) {
      mbar_init(kv_full, 1);
      for (int s = 0; s < C::ST; ++s) {
        mbar_init(&qdo_full[s], 1);
        mbar_init(&qdo_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) mbar_init(&sds_empty[s], 1);
      mbar_init(s_full, 1);
      mbar_init(s_read, 8);
      for (int q = 0; q < 2; ++q) {
        mbar_init(&p_full[q], 8);
        mbar_init(&p_empty[q], 1 + 4);  // the dV MMA (commit) + the tile's four dS warps (P^T in registers)
        mbar_init(&dp_full[q], 1);
        mbar_init(&dp_read[q], 4);
        mbar_init(&ds_full[q], 4);
      }
      mbar_init(dq_full, 1);
      mbar_init(dq_empty, 4);
      mbar_init(acc_full, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(kv_full, 2 * C::kTileBytes);
      tma_load_2d(sK, &P.tk, kv_full, col0, kv_row0);
      tma_load_2d(sV, &P.tv, kv_full, col0, kv_row0);
      for (int i = 0; i < (P.dry == 2 ? 2 : P.n_q); ++i) {
        const int st = i % C::ST;
        mbar_wait(&qdo_empty[st], ((i / C::ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], C::kStageBytes);
        tma_load_2d(sQ(st), &P.tq, &qdo_full[st], col0, q_row_base + i * kTile);
        tma_load_2d(sdO(st), &P.tdo, &qdo_full[st], col0, q_row_base + i * kTile);
        bulk_load_1d(sLse(st), P.lse + stat0 + i * kTile, kTile * 4, &qdo_full[st]);
        bulk_load_1d(sD(st), P.D + stat0 + i * kTile, kTile * 4, &qdo_full[st]);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_ss = make_idesc_bf16_f32(kTile, kTile, false, false);  // [1], [2]
    constexpr uint32_t idesc_ts = make_idesc_bf16_f32(kTile, HD, false, true);      // [3], [4]
    constexpr uint32_t idesc_dq = make_idesc_bf16_f32(kTile, HD, true, true);       // [5]
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
    auto mma_ss = [&](uint32_t d, uint32_t a_base, uint32_t b_base) {  // K-major x K-major over hd = 64
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_bf16(d, make_sw128_desc(a_base + k * 32, 16, 1024), make_sw128_desc(b_base + k * 32, 16, 1024), idesc_ss,
                  k > 0 ? 1u : 0u);
    };
    mbar_wait(kv_full, 0);
    mbar_wait(&qdo_full[0], 0);
    tc_fence_after();
    if (elect_one()) {
      mma_ss(tmem + C::tS, k_base, smem_u32(sQ(0)));
      umma_commit(s_full);
      mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(0)));
      umma_commit(&dp_full[0]);
    }
    __syncwarp();
    for (int i = 0; i < P.n_q; ++i) {
      const int st = i % C::ST;
      const uint32_t ph = i & 1;
      const bool more = i + 1 < P.n_q;
      const int st1 = (i + 1) % C::ST;
      if (more) {
        mbar_wait(s_read, ph);  // the P warps hold S^T_i: the block may take S^T_{i+1}
        if (P.dry != 2 || i + 1 < 2) mbar_wait(&qdo_full[st1], ((i + 1) / C::ST) & 1);
        tc_fence_after();
        if (elect_one()) {
          mma_ss(tmem + C::tS, k_base, smem_u32(sQ(st1)));  // [1]_{i+1}
          umma_commit(s_full);
        }
        __syncwarp();
      }
      const int par = i & 1;
      const uint32_t ph2 = (i >> 1) & 1;
      SSTAMP(7);
      mbar_wait(&p_full[par], ph2);
      SSTAMP(8);
      tc_fence_after();
      if (elect_one()) {  // [3] dV += P^T dO: A = P^T pairs, queries [64g, +64) at tP + [32g, +32)
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + C::tdV, tmem + C::tP + (k >> 2) * 32 + (k & 3) * 8,
                       make_sw128_desc(smem_u32(sdO(st)) + k * 2048, kTile * 128, 1024), idesc_ts,
                       (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&p_empty[par]);
      }
      __syncwarp();
      if (more) {
        mbar_wait(&dp_read[par], ph2);  // the dS warps hold dP^T_i
        SSTAMP(9);
        tc_fence_after();
        if (elect_one()) {
          mma_ss(tmem + C::tdP, v_base, smem_u32(sdO(st1)));  // [2]_{i+1}
          umma_commit(&dp_full[par ^ 1]);
        }
        __syncwarp();
      }
      mbar_wait(&ds_full[par], ph2);
      SSTAMP(10);
      tc_fence_after();
      const uint32_t ds_base = smem_u32(sdS + (i & 1) * C::kDsBytes);
      if (elect_one()) {
        // [4] dK += dS^T Q: A = dS^T K-major in shared memory (chunk g = queries [64g, +64), 128 B rows)
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16(tmem + C::tdK, make_sw128_desc(ds_base + (k >> 2) * (kTile * 128) + (k & 3) * 32, 16, 1024),
                    make_sw128_desc(smem_u32(sQ(st)) + k * 2048, kTile * 128, 1024), idesc_ts,
                    (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&qdo_empty[st]);
      }
      __syncwarp();
      if (i >= 1) {
        mbar_wait(dq_empty, (i - 1) & 1);  // the reduce warps have drained dQ_{i-1}
        tc_fence_after();
      }
      SSTAMP(11);
      if (elect_one()) {
        // [5] dQ_i = dS K: A = dS MN-major (the same tile), B = K MN-major
#pragma unroll
        for (int k = 0; k < kTile / 16; ++k)
          umma_bf16(tmem + C::tdQ, make_sw128_desc(ds_base + k * 2048, kTile * 128, 1024),
                    make_sw128_desc(k_base + k * 2048, kTile * 128, 1024), idesc_dq, k > 0 ? 1u : 0u);
        umma_commit(dq_full);
        umma_commit(&sds_empty[i & 1]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
  } else if (warp < 10) {
    // ---------------------------------------------------------------- P warps 2..9
    const uint32_t g = (warp - 2) >> 2;
    const uint32_t q4 = warp & 3;
    const uint32_t lane_addr = (q4 * 32) << 16;
    const float2 c2 = make_float2(P.c, P.c);
    for (int i = 0; i < P.n_q; ++i) {
      const int st = i % C::ST;
      const uint32_t lse_a = smem_u32(sLse(st)) + g * 256;
      if (P.dry != 2 || i < 2) mbar_wait(&qdo_full[st], (i / C::ST) & 1);  // lse of this query tile is resident
      mbar_wait(s_full, i & 1);
      if (q4 == 2) SSTAMP(g);
      tc_fence_after();
      if (P.dry) {
        __syncwarp();
        if (lane == 0) mbar_arrive(s_read);
        if (i >= 1) mbar_wait(&p_empty[(i - 1) & 1], ((i - 1) >> 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i & 1]);
        continue;
      }
      // two 32-column halves (register budget: 22 warps share the register file)
      uint32_t pk[2][16];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t sv[32];
        tmem_ld_32x32b_x32(tmem + C::tS + lane_addr + g * 64 + hh * 32, sv);
        tmem_ld_wait();
        if (hh == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_read);
        }
#pragma unroll
        for (int m = 0; m < 32; m += 4) {
          const float4 l4 = (P.diag & 4) ? make_float4(__int_as_float(lse_a), 1.f, 2.f, 3.f)
                                         : ld_shared_f4(lse_a + (hh * 32 + m) * 4);
          const float2 x01 = ffma2(make_float2(__uint_as_float(sv[m]), __uint_as_float(sv[m + 1])), c2,
                                   make_float2(-l4.x, -l4.y));
          const float2 x23 = ffma2(make_float2(__uint_as_float(sv[m + 2]), __uint_as_float(sv[m + 3])), c2,
                                   make_float2(-l4.z, -l4.w));
          pk[hh][m / 2] = pack_bf16(ex2_approx(x01.x), ex2_approx(x01.y));
          pk[hh][m / 2 + 1] = pack_bf16(ex2_approx(x23.x), ex2_approx(x23.y));
        }
      }
      if (i >= 1) {
        mbar_wait(&p_empty[(i - 1) & 1], ((i - 1) >> 1) & 1);  // the dV MMA and the dS warps are done with P^T_{i-1}
        tc_fence_after();
      }
      tmem_st_32x32b_x16(tmem + C::tP + lane_addr + g * 32, pk[0]);
      tmem_st_32x32b_x16(tmem + C::tP + lane_addr + g * 32 + 16, pk[1]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i & 1]);
      if (q4 == 2) SSTAMP(2 + g);
    }
    // ---------------------------------------------------------------- dK / dV epilogue (group 0: dV, 1: dK)
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t row = q4 * 32 + lane;
    const uint32_t tcol = g == 0 ? C::tdV : C::tdK;
    const float sc = g == 0 ? 1.f : P.dk_scale;
    __nv_bfloat16* out = g == 0 ? P.dv + (long long)(kv_row0 + row) * P.lddv + col0
                                : P.dk + (long long)(kv_row0 + row) * P.lddk + col0;
#pragma unroll
    for (int cc = 0; cc < HD / 32; ++cc) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tmem + tcol + lane_addr + cc * 32, o);
      tmem_ld_wait();
      uint32_t ok[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) ok[j] = pack_bf16(__uint_as_float(o[2 * j]) * sc, __uint_as_float(o[2 * j + 1]) * sc);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_global_v4(out + cc * 32 + v * 8, make_uint4(ok[4 * v], ok[4 * v + 1], ok[4 * v + 2], ok[4 * v + 3]));
    }
  } else if (warp < 18) {
    // ---------------------------------------------------------------- dS warps 10..17 (group = tile parity)
    const int grp = (int)(warp - 10) >> 2;
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // key row within the tile == TMEM lane
    const uint32_t lane_addr = (q4 * 32) << 16;
    for (int i = grp; i < P.n_q; i += 2) {
      const int st = i % C::ST;
      const int par = i & 1;  // == grp
      const uint32_t ph2 = (i >> 1) & 1;
      const uint32_t d_a = smem_u32(sD(st));
      if (P.dry != 2 || i < 2) mbar_wait(&qdo_full[st], (i / C::ST) & 1);  // D of this query tile is resident
      mbar_wait(&dp_full[par], ph2);
      mbar_wait(&p_full[par], ph2);
      tc_fence_after();
      if (i >= 2) mbar_wait(&sds_empty[par], ((i >> 1) - 1) & 1);  // dQ_{i-2} has read this dS buffer
      if (q4 == 2 && grp == 0) SSTAMP(4);
      if (P.dry) {
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&dp_read[par]);
          mbar_arrive(&p_empty[par]);
          mbar_arrive(&ds_full[par]);
        }
        continue;
      }
      const uint32_t ds_row0 = smem_u32(sdS + par * C::kDsBytes) + row * 128;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {  // 32 queries per chunk
        uint32_t dp[32], pp[16];
        tmem_ld_32x32b_x32(tmem + C::tdP + lane_addr + cc * 32, dp);
        tmem_ld_32x32b_x16(tmem + C::tP + lane_addr + cc * 16, pp);
        tmem_ld_wait();
        if (cc == 3) {  // dP^T_i and P^T_i are in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&dp_read[par]);
            mbar_arrive(&p_empty[par]);
          }
        }
        const uint32_t base = ds_row0 + (cc >> 1) * (kTile * 128);
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // 8 queries per 16-byte unit
          uint32_t ds[4];
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            const int mm = u * 8 + j;  // column within the chunk
            const float4 d4 = (P.diag & 4) ? make_float4(__int_as_float(d_a), 1.f, 2.f, 3.f)
                                           : ld_shared_f4(d_a + (cc * 32 + mm) * 4);
            const uint32_t p01 = pp[mm / 2], p23 = pp[mm / 2 + 1];
            const float2 a01 = fmul2(make_float2(bf16_lo(p01), bf16_hi(p01)),
                                     fadd2(make_float2(__uint_as_float(dp[mm]), __uint_as_float(dp[mm + 1])),
                                           make_float2(-d4.x, -d4.y)));
            const float2 a23 = fmul2(make_float2(bf16_lo(p23), bf16_hi(p23)),
                                     fadd2(make_float2(__uint_as_float(dp[mm + 2]), __uint_as_float(dp[mm + 3])),
                                           make_float2(-d4.z, -d4.w)));
            ds[j / 2] = pack_bf16(a01.x, a01.y);
            ds[j / 2 + 1] = pack_bf16(a23.x, a23.y);
          }
          const uint32_t unit = (cc & 1) * 4 + u;
          if (P.diag & 1) {
            if ((ds[0] ^ ds[1] ^ ds[2] ^ ds[3]) == 0x12345678u) st_shared_v4(base, 0, 0, 0, 0);
          } else {
            st_shared_v4(base + ((unit ^ (row & 7)) << 4), ds[0], ds[1], ds[2], ds[3]);
          }
        }
      }
      if (!(P.diag & 2)) fence_proxy_async_smem();  // the stores, for the dK / dQ MMAs (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[par]);
      if (q4 == 2 && grp == 0) SSTAMP(5);
    }
  } else {
    // ---------------------------------------------------------------- dQ reduce warps 18..21
    const uint32_t q4 = warp & 3;
    const uint32_t row = q4 * 32 + lane;  // query row within the tile
    const uint32_t lane_addr = (q4 * 32) << 16;
    const bool issuer = (warp == 18 && lane == 0);
    for (int i = 0; i < P.n_q; ++i) {
      mbar_wait(dq_full, i & 1);
      if (q4 == 2) SSTAMP(13);
      tc_fence_after();
      if (P.dry) {
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_empty);
        continue;
      }
#pragma unroll
      for (int bx = 0; bx < 2; ++bx) {  // one 32-column box at a time through the 16 KB staging tile
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + C::tdQ + lane_addr + bx * 32, o);
        tmem_ld_wait();
        if (bx == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_empty);
        }
        if (issuer) bulk_wait_read<0>();  // the previous box's reduce has read the staging tile
        named_bar_sync(1, 128);
        const uint32_t base = smem_u32(sdQ) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(base + ((u ^ (row & 7)) << 4), o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (issuer) {
          tma_reduce_add_2d(&P.tdq, sdQ, col0 + 32 * bx, q_row_base + i * kTile);
          bulk_commit();
        }
      }
    }
    if (issuer) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
#undef SSTAMP
}

// D[b, h, s] = sum_hd dO o O (fp32) per (row, head); zero the fp32 dQ accumulator. One warp per row.
template <int HD>
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, long long ldo,
                                     const __nv_bfloat16* __restrict__ dO, long long lddo, float* __restrict__ D,
                                     float* __restrict__ dq_acc, long long ldacc, int rows, int s, int h) {
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  constexpr int kLanesPerHead = HD / 8;
  for (int r = blockIdx.x * warps + threadIdx.x / 32; r < rows; r += gridDim.x * warps) {
    const int bi = r / s, si = r - bi * s;
    for (int c = lane * 8; c < h * HD; c += 32 * 8) {
      const uint4 a = *reinterpret_cast<const uint4*>(o + (long long)r * ldo + c);
      const uint4 g = *reinterpret_cast<const uint4*>(dO + (long long)r * lddo + c);
      float acc = bf16_lo(a.x) * bf16_lo(g.x) + bf16_hi(a.x) * bf16_hi(g.x);
      acc = fmaf(bf16_lo(a.y), bf16_lo(g.y), acc);
      acc = fmaf(bf16_hi(a.y), bf16_hi(g.y), acc);
      acc = fmaf(bf16_lo(a.z), bf16_lo(g.z), acc);
      acc = fmaf(bf16_hi(a.z), bf16_hi(g.z), acc);
      acc = fmaf(bf16_lo(a.w), bf16_lo(g.w), acc);
      acc = fmaf(bf16_hi(a.w), bf16_hi(g.w), acc);
#pragma unroll
      for (int off = kLanesPerHead / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if ((lane % kLanesPerHead) == 0) D[((long long)bi * h + c / HD) * s + si] = acc;
      float4* z = reinterpret_cast<float4*>(dq_acc + (long long)r * ldacc + c);
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// dq = bf16(scale * dq_acc)
__global__ void attn_bwd_dq_kernel(const float* __restrict__ acc, long long ldacc, __nv_bfloat16* __restrict__ dq,
                                   long long lddq, int rows, int width, float scale) {
  const int per_row = width / 8;
  const long long n = (long long)rows * per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row), c = (int)(i - (long long)r * per_row) * 8;
    const float4 a = *reinterpret_cast<const float4*>(acc + (long long)r * ldacc + c);
    const float4 b = *reinterpret_cast<const float4*>(acc + (long long)r * ldacc + c + 4);
    *reinterpret_cast<uint4*>(dq + (long long)r * lddq + c) =
        make_uint4(pack_bf16(a.x * scale, a.y * scale), pack_bf16(a.z * scale, a.w * scale),
                   pack_bf16(b.x * scale, b.y * scale), pack_bf16(b.z * scale, b.w * scale));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// [rows, width] bf16 row-major with row stride ld elements; 64 x 128 boxes, 128B swizzle.
int head_tile_map(CUtensorMap* m, const void* ptr, int rows, int width, long long ld) {
  auto enc = encode_fn();
  if (!enc) return BTP_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, kTile};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? BTP_OK : BTP_ERR_ALIGNMENT;
}

// fp32 [rows, width] with row stride ld elements; 32 x 128 boxes (128 B rows), 128B swizzle.
int f32_tile_map(CUtensorMap* m, const void* ptr, int rows, int width, long long ld) {
  auto enc = encode_fn();
  if (!enc) return BTP_ERR_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, kTile};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? BTP_OK : BTP_ERR_ALIGNMENT;
}

static int g_fwd_poly = 2;     // every n-th exp2 pair on the FMA pipe (0: all on the MUFU)
static int g_fwd_dry = 0;      // diagnostics: handshake-only softmax in the split-row kernels (wrong results)
static int g_fwd_variant = 4;  // 4: two query tiles per CTA (s % 256), 3: split rows single S, 2 / 1: split rows
                               // double-buffered with 4 / 2 key groups (hd 128: 2), 0: attn_fwd_kernel;
                               // hd 64, s % 256: 5 two query tiles with P apart from S, 6 the same, split rows

template <int HD, int ST, int kPoly>
int launch_fwd_poly(const FwdParams& P, int b, cudaStream_t stream) {
  using C = FwdCfg<HD, ST>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd_kernel<HD, ST, kPoly>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmem) != cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  dim3 grid(P.s / kTile, P.h, b);
  attn_fwd_kernel<HD, ST, kPoly><<<grid, C::kThreads, C::kSmem, stream>>>(P);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

template <int HD, int ST>
int launch_bwd(const BwdParams& P, int b, cudaStream_t stream) {
  using C = BwdCfg<HD, ST>;
  static_assert(C::kSmem <= 232448, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd_kernel<HD, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  dim3 grid(P.s / kTile, P.h, b);
  attn_bwd_kernel<HD, ST><<<grid, C::kThreads, C::kSmem, stream>>>(P);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

static int g_bwd_poly = 2;  // every n-th group of 4 exp2s in the backward's P phase: 2 on the FMA pipe (0: none);
                            // 2 (default): 1748 vs 1819 us median under sustained load, same cold (r02_bwd_poly_ab.log)

static int g_bwd_persist = 1;  // 1 (default): persistent hd-64 backward (one CTA per SM walking the work items;
                               // 1552 vs 1629 us at the bench shape, scripts/microbench/attn_bwd_variants.py 7)

template <bool kTrace, int kPoly, bool kPk>
int launch_bwd64_t(const BwdParams& P, int b, cudaStream_t stream) {
  using C = Bwd64Cfg;
  static_assert(C::kSmem <= 232448, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd64_kernel<kTrace, kPoly, kPk>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmem) != cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  BwdParams Q = P;
  Q.n_items = P.n_q * P.h * b;
  const int nsm = num_sms_cached();
  const int grid = g_bwd_persist && Q.n_items > nsm ? nsm : Q.n_items;
  attn_bwd64_kernel<kTrace, kPoly, kPk><<<grid, C::kThreads, C::kSmem, stream>>>(Q);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

template <bool kTrace, bool kPk>
int launch_bwd64_p(const BwdParams& P, int b, cudaStream_t stream) {
  switch (g_bwd_poly) {
    case 1: return launch_bwd64_t<kTrace, 1, kPk>(P, b, stream);
    case 2: return launch_bwd64_t<kTrace, 2, kPk>(P, b, stream);
    case 4: return launch_bwd64_t<kTrace, 4, kPk>(P, b, stream);
    default: return launch_bwd64_t<kTrace, 0, kPk>(P, b, stream);
  }
}

static int g_bwd_variant = 0;  // 1: split-role hd-64 kernel (attn_bwd64s_kernel), 0: attn_bwd64_kernel (default),
                               // 2: attn_bwd64_kernel with the packed-P dS phase (kPk)
static int g_bwd_dry = 0;      // diagnostics: handshakes only in the split-role kernel (wrong results)
static int g_bwd_diag = 0;     // diagnostics: BwdParams::diag bits (wrong results)

int launch_bwd64s(const BwdParams& P, int b, cudaStream_t stream) {
  using C = Bwd64sCfg;
  static_assert(C::kSmem <= 232448, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd64s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  dim3 grid(P.s / kTile, P.h, b);
  BwdParams Q = P;
  Q.dry = g_bwd_dry;
  Q.diag = g_bwd_diag;
  attn_bwd64s_kernel<<<grid, C::kThreads, C::kSmem, stream>>>(Q);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int launch_bwd64(const BwdParams& P, int b, cudaStream_t stream) {
  if (g_bwd_variant == 1) return launch_bwd64s(P, b, stream);
  if (g_bwd_variant == 2)
    return P.trace != nullptr ? launch_bwd64_p<true, true>(P, b, stream) : launch_bwd64_p<false, true>(P, b, stream);
  return P.trace != nullptr ? launch_bwd64_p<true, false>(P, b, stream) : launch_bwd64_p<false, false>(P, b, stream);
}

template <int HD, int ST, int kPoly, int kSplit, int kSBuf = 2, int kQT = 1>
int launch_fwd2_poly(const FwdParams& P, int b, cudaStream_t stream) {
  using C = Fwd2Cfg<HD, ST, kSplit, kSBuf, kQT>;
  static_assert(C::kSmem <= 232448 / C::kCtasPerSm, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd2_kernel<HD, ST, kPoly, kSplit, kSBuf, kQT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) != cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  dim3 grid(P.s / (kTile * kQT), P.h, b);
  FwdParams Q = P;
  Q.dry = g_fwd_dry;
  attn_fwd2_kernel<HD, ST, kPoly, kSplit, kSBuf, kQT><<<grid, C::kThreads, C::kSmem, stream>>>(Q);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

template <int HD, int ST, int kSplit, int kSBuf = 2, int kQT = 1>
int launch_fwd2(const FwdParams& P, int b, cudaStream_t stream) {
  switch (g_fwd_poly) {
    case 0: return launch_fwd2_poly<HD, ST, 0, kSplit, kSBuf, kQT>(P, b, stream);
    case 2: return launch_fwd2_poly<HD, ST, 2, kSplit, kSBuf, kQT>(P, b, stream);
    case 3: return launch_fwd2_poly<HD, ST, 3, kSplit, kSBuf, kQT>(P, b, stream);
    case 5: return launch_fwd2_poly<HD, ST, 5, kSplit, kSBuf, kQT>(P, b, stream);
    default: return launch_fwd2_poly<HD, ST, 4, kSplit, kSBuf, kQT>(P, b, stream);
  }
}

template <int ST, int kPoly, int kHalves>
int launch_fwd3_poly(const FwdParams& P, int b, cudaStream_t stream) {
  using C = Fwd3Cfg<ST, kHalves>;
  static_assert(C::kSmem <= 232448, "shared memory budget");
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd3_kernel<ST, kPoly, kHalves>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmem) != cudaSuccess)
      return BTP_ERR_CUDA;
    configured = true;
  }
  dim3 grid(P.s / (2 * kTile), P.h, b);
  attn_fwd3_kernel<ST, kPoly, kHalves><<<grid, C::kThreads, C::kSmem, stream>>>(P);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

template <int ST, int kHalves>
int launch_fwd3(const FwdParams& P, int b, cudaStream_t stream) {
  switch (g_fwd_poly) {
    case 0: return launch_fwd3_poly<ST, 0, kHalves>(P, b, stream);
    case 2: return launch_fwd3_poly<ST, 2, kHalves>(P, b, stream);
    case 3: return launch_fwd3_poly<ST, 3, kHalves>(P, b, stream);
    case 5: return launch_fwd3_poly<ST, 5, kHalves>(P, b, stream);
    default: return launch_fwd3_poly<ST, 4, kHalves>(P, b, stream);
  }
}

template <int HD, int ST>
int launch_fwd(const FwdParams& P, int b, cudaStream_t stream) {
  switch (g_fwd_poly) {
    case 0: return launch_fwd_poly<HD, ST, 0>(P, b, stream);
    case 2: return launch_fwd_poly<HD, ST, 2>(P, b, stream);
    case 3: return launch_fwd_poly<HD, ST, 3>(P, b, stream);
    case 5: return launch_fwd_poly<HD, ST, 5>(P, b, stream);
    default: return launch_fwd_poly<HD, ST, 4>(P, b, stream);
  }
}

}  // namespace

int attn_tune(int key, int value) {
  int* slot = key == 0   ? &g_fwd_poly
              : key == 1 ? &g_fwd_variant
              : key == 2 ? &g_bwd_poly
              : key == 3 ? &g_bwd_variant
              : key == 4 ? &g_bwd_dry
              : key == 5 ? &g_bwd_diag
              : key == 6 ? &g_fwd_dry
              : key == 7 ? &g_bwd_persist
                         : nullptr;
  if (slot == nullptr) return -1;
  const int prev = *slot;
  if (value >= 0) *slot = value;
  return prev;
}

int attn_fwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, void* o,
             long long ldo, float* lse, int b, int s, int h, int hd, cudaStream_t stream, long long* trace) {
  if (b <= 0 || s <= 0 || h <= 0) return BTP_ERR_DIM;
  if (s % kTile != 0 || (hd != 64 && hd != 128)) return BTP_ERR_DIM;
  const long long width = (long long)h * hd;
  if (ldq < width || ldk < width || ldv < width || ldo < width) return BTP_ERR_DIM;
  auto mis = [](const void* p, long long ld) {
    return (reinterpret_cast<uintptr_t>(p) & 15) != 0 || (ld * 2) % 16 != 0;
  };
  if (mis(q, ldq) || mis(k, ldk) || mis(v, ldv) || mis(o, ldo) || lse == nullptr) return BTP_ERR_ALIGNMENT;
  FwdParams P{};
  const int rows = b * s;
  int rc;
  if ((rc = head_tile_map(&P.tq, q, rows, (int)width, ldq)) != BTP_OK) return rc;
  if ((rc = head_tile_map(&P.tk, k, rows, (int)width, ldk)) != BTP_OK) return rc;
  if ((rc = head_tile_map(&P.tv, v, rows, (int)width, ldv)) != BTP_OK) return rc;
  P.o = static_cast<__nv_bfloat16*>(o);
  P.ldo = ldo;
  P.lse = lse;
  P.s = s;
  P.h = h;
  P.n_kv = s / kTile;
  P.c = 1.4426950408889634f / sqrtf((float)hd);
  P.trace = trace;
  if (g_fwd_variant == 5 && s % 256 == 0 && hd == 64) return launch_fwd3<4, 1>(P, b, stream);
  if (g_fwd_variant == 6 && s % 256 == 0 && hd == 64) return launch_fwd3<4, 2>(P, b, stream);
  if (g_fwd_variant >= 4 && s % 256 == 0)
    return hd == 64 ? launch_fwd2<64, 3, 2, 1, 2>(P, b, stream) : launch_fwd2<128, 2, 1, 1, 2>(P, b, stream);
  if (g_fwd_variant == 3 && hd == 64) return launch_fwd2<64, 2, 2, 1>(P, b, stream);
  if (g_fwd_variant == 2 && hd == 64) return launch_fwd2<64, 3, 4>(P, b, stream);
  if (g_fwd_variant >= 1) return hd == 64 ? launch_fwd2<64, 3, 2>(P, b, stream) : launch_fwd2<128, 2, 2>(P, b, stream);
  return hd == 64 ? launch_fwd<64, 2>(P, b, stream) : launch_fwd<128, 1>(P, b, stream);
}

int attn_bwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, const void* o,
             long long ldo, const void* dO, long long lddo, const float* lse, float* D, float* dq_acc,
             long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv, long long lddv, int b,
             int s, int h, int hd, cudaStream_t stream, long long* trace) {
  if (b <= 0 || s <= 0 || h <= 0) return BTP_ERR_DIM;
  if (s % kTile != 0 || (hd != 64 && hd != 128)) return BTP_ERR_DIM;
  const long long width = (long long)h * hd;
  if (ldq < width || ldk < width || ldv < width || ldo < width || lddo < width || ldacc < width || lddq < width ||
      lddk < width || lddv < width)
    return BTP_ERR_DIM;
  auto mis = [](const void* p, long long ld) {
    return (reinterpret_cast<uintptr_t>(p) & 15) != 0 || (ld * 2) % 16 != 0;
  };
  if (mis(q, ldq) || mis(k, ldk) || mis(v, ldv) || mis(o, ldo) || mis(dO, lddo) || mis(dq, lddq) || mis(dk, lddk) ||
      mis(dv, lddv) || mis(dq_acc, 2 * ldacc) || lse == nullptr || D == nullptr)
    return BTP_ERR_ALIGNMENT;
  if ((reinterpret_cast<uintptr_t>(lse) & 15) || (reinterpret_cast<uintptr_t>(D) & 15)) return BTP_ERR_ALIGNMENT;
  const int rows = b * s;
  const int nsm = num_sms_cached();
  if (hd == 64)
    attn_bwd_prep_kernel<64><<<nsm * 8, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(o), ldo,
                                                          static_cast<const __nv_bfloat16*>(dO), lddo, D, dq_acc,
                                                          ldacc, rows, s, h);
  else
    attn_bwd_prep_kernel<128><<<nsm * 8, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(o), ldo,
                                                           static_cast<const __nv_bfloat16*>(dO), lddo, D, dq_acc,
                                                           ldacc, rows, s, h);
  BwdParams P{};
  int rc;
  if ((rc = head_tile_map(&P.tq, q, rows, (int)width, ldq)) != BTP_OK) return rc;
  if ((rc = head_tile_map(&P.tk, k, rows, (int)width, ldk)) != BTP_OK) return rc;
  if ((rc = head_tile_map(&P.tv, v, rows, (int)width, ldv)) != BTP_OK) return rc;
  if ((rc = head_tile_map(&P.tdo, dO, rows, (int)width, lddo)) != BTP_OK) return rc;
  if ((rc = f32_tile_map(&P.tdq, dq_acc, rows, (int)width, ldacc)) != BTP_OK) return rc;
  P.lse = lse;
  P.D = D;
  P.dq_acc = dq_acc;
  P.ldacc = ldacc;
  P.dk = static_cast<__nv_bfloat16*>(dk);
  P.lddk = lddk;
  P.dv = static_cast<__nv_bfloat16*>(dv);
  P.lddv = lddv;
  P.s = s;
  P.h = h;
  P.n_q = s / kTile;
  P.dk_scale = 1.f / sqrtf((float)hd);
  P.c = 1.4426950408889634f * P.dk_scale;
  P.trace = trace;
  rc = hd == 64 ? launch_bwd64(P, b, stream) : launch_bwd<128, 2>(P, b, stream);
  if (rc != BTP_OK) return rc;
  attn_bwd_dq_kernel<<<nsm * 8, 256, 0, stream>>>(dq_acc, ldacc, static_cast<__nv_bfloat16*>(dq), lddq, rows,
                                                  (int)width, P.dk_scale);
  return cudaGetLastError() == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

}  // namespace btp
