// extern "C" boundary of libbtp.so: argument marshalling only; every entry point forwards
// to the kernels in gemm.cu / gemm_f32.cu / rowops.cu on the caller's stream. See include/btp.h.
// The *_f32 twins take fp32 activations (parity mode); everything else is bf16.
#include <cuda_runtime.h>

#include "btp_internal.h"

namespace btp {
int num_sms_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}
}  // namespace btp

#define ST(s) static_cast<cudaStream_t>(s)

// Defines NAME (bf16) and NAME_f32 (fp32) for a row kernel whose last two internal args are (stream, f32).
#define BTP_PAIR(NAME, IMPL, PARAMS, ARGS)                                             \
  int NAME PARAMS { return btp::IMPL ARGS(false); }                                    \
  int NAME##_f32 PARAMS { return btp::IMPL ARGS(true); }

extern "C" {

int btp_gemm(const btp_gemm_problem* problems, int n, int bn_hint, void* stream) {
  return btp::gemm_launch(problems, n, bn_hint, 0, ST(stream));
}

int btp_gemm_scatter(const btp_gemm_problem* problems, int n, int bn_hint, void* const* owners, int n_owners,
                     int rows_per_owner, int width, long long ld, const int* col0, void* stream) {
  if (owners == nullptr || col0 == nullptr) return BTP_ERR_DIM;
  const btp::ScatterSpec sc{n_owners, owners, rows_per_owner, width, ld, col0};
  return btp::gemm_launch_scatter(problems, n, bn_hint, 0, ST(stream), &sc);
}

int btp_attn_fwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, void* o,
                 long long ldo, float* lse, int b, int s, int h, int hd, void* stream) {
  return btp::attn_fwd(q, ldq, k, ldk, v, ldv, o, ldo, lse, b, s, h, hd, ST(stream));
}

int btp_attn_bwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                 const void* o, long long ldo, const void* dO, long long lddo, const float* lse, float* D,
                 float* dq_acc, long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv,
                 long long lddv, int b, int s, int h, int hd, void* stream) {
  return btp::attn_bwd(q, ldq, k, ldk, v, ldv, o, ldo, dO, lddo, lse, D, dq_acc, ldacc, dq, lddq, dk, lddk, dv, lddv,
                       b, s, h, hd, ST(stream));
}

int btp_attn_bwd_trace(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                       const void* o, long long ldo, const void* dO, long long lddo, const float* lse, float* D,
                       float* dq_acc, long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv,
                       long long lddv, int b, int s, int h, int hd, long long* trace, void* stream) {
  return btp::attn_bwd(q, ldq, k, ldk, v, ldv, o, ldo, dO, lddo, lse, D, dq_acc, ldacc, dq, lddq, dk, lddk, dv, lddv,
                       b, s, h, hd, ST(stream), trace);
}

int btp_attn_fwd_trace(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                       void* o, long long ldo, float* lse, int b, int s, int h, int hd, long long* trace, void* stream) {
  return btp::attn_fwd(q, ldq, k, ldk, v, ldv, o, ldo, lse, b, s, h, hd, ST(stream), trace);
}

int btp_attn_tune(int key, int value) { return btp::attn_tune(key, value); }

int btp_gemm_f32(const btp_gemm_problem* problems, int n, void* stream) {
  return btp::gemm_f32_launch(problems, n, ST(stream));
}

#define A_RMSNORM_RESIDUAL(f32) \
  (x, ldx, branch, ldb, x_out, ldo, gamma, n_out, ldn, ss_out, rms_loc_out, rows, width, eps, ST(stream), f32)
BTP_PAIR(btp_rmsnorm_residual, rmsnorm_residual,
         (const void* x, long long ldx, const void* branch, long long ldb, void* x_out, long long ldo,
          const float* gamma, void* n_out, long long ldn, float* ss_out, float* rms_loc_out, int rows, int width,
          float eps, void* stream),
         A_RMSNORM_RESIDUAL)

#define A_RMSNORM_APPLY(f32) (x, ldx, gamma, ss_total, d, eps, n_out, ldn, rms_out, rows, width, ST(stream), f32)
BTP_PAIR(btp_rmsnorm_apply, rmsnorm_apply,
         (const void* x, long long ldx, const float* gamma, const float* ss_total, int d, float eps, void* n_out,
          long long ldn, float* rms_out, int rows, int width, void* stream),
         A_RMSNORM_APPLY)

#define A_FIXUP(f32) (P, ldp, ss_total, d, eps, s_out, z_out, ldz, a_out, lda, rows, r, nproj, variant, ST(stream), f32)
BTP_PAIR(btp_fixup_sigma, fixup_sigma,
         (const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out, void* z_out,
          long long ldz, void* a_out, long long lda, int rows, int r, int nproj, int variant, void* stream),
         A_FIXUP)

int btp_fixup_sigma_f32in(const float* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                          void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj,
                          int variant, void* stream) {
  return btp::fixup_sigma_f32in(P, ldp, ss_total, d, eps, s_out, z_out, ldz, a_out, lda, rows, r, nproj, variant,
                                ST(stream));
}

#define A_SWIGLU(f32) (g, ldg, u, ldu, act, lda, rows, cols, ST(stream), f32)
BTP_PAIR(btp_swiglu, swiglu,
         (const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda, int rows, int cols,
          void* stream),
         A_SWIGLU)

#define A_SWIGLU_BWD(f32) (g, ldg, u, ldu, dact, ldda, dg, lddg, du, lddu, rows, cols, ST(stream), f32)
BTP_PAIR(btp_swiglu_bwd, swiglu_bwd,
         (const void* g, long long ldg, const void* u, long long ldu, const void* dact, long long ldda, void* dg,
          long long lddg, void* du, long long lddu, int rows, int cols, void* stream),
         A_SWIGLU_BWD)

#define A_FIXUP_BWD(f32) (z, ldz, da, ldda, s, d, dP, lddp, dss, rows, r, nproj, variant, ST(stream), f32)
BTP_PAIR(btp_fixup_sigma_bwd, fixup_sigma_bwd,
         (const void* z, long long ldz, const void* da, long long ldda, const float* s, int d, void* dP,
          long long lddp, float* dss, int rows, int r, int nproj, int variant, void* stream),
         A_FIXUP_BWD)

#define A_NORM_BWD(f32) \
  (dh, lddh, x, ldx, gamma, dss, dres, ldr, dx, lddx, dgamma_partial, max_blocks, nblk, rows, width, ST(stream), f32)
BTP_PAIR(btp_rmsnorm_bwd, rmsnorm_bwd,
         (const void* dh, long long lddh, const void* x, long long ldx, const float* gamma, const float* dss,
          const void* dres, long long ldr, void* dx, long long lddx, float* dgamma_partial, int max_blocks, int* nblk,
          int rows, int width, void* stream),
         A_NORM_BWD)

#define A_NORM_PREP(f32) (dn, lddn, x, ldx, gamma, s, dh, lddh, dss, rows, width, ST(stream), f32)
BTP_PAIR(btp_rmsnorm_bwd_prep, rmsnorm_bwd_prep,
         (const void* dn, long long lddn, const void* x, long long ldx, const float* gamma, const float* s, void* dh,
          long long lddh, float* dss, int rows, int width, void* stream),
         A_NORM_PREP)

#define A_ADD(f32) (a, lda, b, ldb, out, ldo, rows, cols, ST(stream), f32)
BTP_PAIR(btp_add, add,
         (const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows, int cols,
          void* stream),
         A_ADD)

#define A_DOT(f32) (a, lda, b, ldb, rows, cols, partial, max_blocks, nblk, ST(stream), f32)
BTP_PAIR(btp_dot, dot,
         (const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
          int max_blocks, int* nblk, void* stream),
         A_DOT)

#define A_ADAMW(f32) (master, m, v, g, work, n, lr, b1, b2, eps, wd, step, step_dev, ST(stream), f32)
BTP_PAIR(btp_adamw, adamw,
         (float* master, float* m, float* v, const float* g, void* work, long long n, float lr, float b1, float b2,
          float eps, float wd, int step, const int* step_dev, void* stream),
         A_ADAMW)

#define A_EMB_FWD(f32) (ids, table, ldt, vocab, col0, out, ldo, rows, width, bad, ST(stream), f32)
BTP_PAIR(btp_embedding_fwd, embedding_fwd,
         (const int* ids, const void* table, long long ldt, int vocab, int col0, void* out, long long ldo, int rows,
          int width, int* bad, void* stream),
         A_EMB_FWD)

#define A_EMB_BWD(f32) (ids, dx, lddx, vocab, dtable, ldg, rows, width, ST(stream), f32)
BTP_PAIR(btp_embedding_bwd, embedding_bwd,
         (const int* ids, const void* dx, long long lddx, int vocab, float* dtable, long long ldg, int rows, int width,
          void* stream),
         A_EMB_BWD)

#define A_XENT(f32) (logits, ldl, targets, vocab, loss_rows, dlogits, ldd, rows, scale, ST(stream), f32)
BTP_PAIR(btp_cross_entropy, cross_entropy,
         (const void* logits, long long ldl, const int* targets, int vocab, float* loss_rows, void* dlogits,
          long long ldd, int rows, float scale, void* stream),
         A_XENT)

int btp_peer_signal(unsigned int* const* peer_flags, unsigned int* epoch, int slot, int rank, int tp, void* stream) {
  return btp::peer_signal(peer_flags, epoch, slot, rank, tp, ST(stream));
}

int btp_peer_wait(const unsigned int* flags, const unsigned int* epoch, int slot, int tp, void* stream) {
  return btp::peer_wait(flags, epoch, slot, tp, ST(stream));
}

int btp_peer_boundary_fwd(const void* const* P_peers, const float* const* ss_peers, int tp, int rank, int T, int W,
                          int r, int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                          void* stream) {
  return btp::peer_boundary_fwd(P_peers, ss_peers, tp, rank, T, W, r, variant, d, eps, z_own, s_own, a_peers,
                                ST(stream));
}

int btp_peer_boundary_bwd(const void* const* da_peers, int tp, int rank, int T, int W, int r, int variant, int d,
                          const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                          void* stream) {
  return btp::peer_boundary_bwd(da_peers, tp, rank, T, W, r, variant, d, z_own, s_own, dP_peers, dss_peers,
                                ST(stream));
}

int btp_peer_boundary_fwd_local(void* R_own, const float* const* ss_peers, int tp, int rank, int T, int W, int r,
                                int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                                void* stream) {
  if (R_own == nullptr) return BTP_ERR_DIM;
  return btp::peer_boundary_fwd(nullptr, ss_peers, tp, rank, T, W, r, variant, d, eps, z_own, s_own, a_peers,
                                ST(stream), R_own);
}

int btp_peer_boundary_bwd_local(void* R_own, int tp, int rank, int T, int W, int r, int variant, int d,
                                const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                                void* stream) {
  if (R_own == nullptr) return BTP_ERR_DIM;
  return btp::peer_boundary_bwd(nullptr, tp, rank, T, W, r, variant, d, z_own, s_own, dP_peers, dss_peers,
                                ST(stream), R_own);
}

int btp_peer_boundary_fwd_nvls(const void* P_mc, const float* ss_mc, int tp, int rank, int T, int W, int r,
                               int variant, int d, float eps, void* z_own, float* s_own, void* a_mc, void* stream) {
  return btp::peer_boundary_fwd_nvls(P_mc, ss_mc, tp, rank, T, W, r, variant, d, eps, z_own, s_own, a_mc, ST(stream));
}

int btp_peer_boundary_bwd_nvls(const void* dA_mc, int tp, int rank, int T, int W, int r, int variant, int d,
                               const void* z_own, const float* s_own, void* dP_mc, float* dss_mc, void* stream) {
  return btp::peer_boundary_bwd_nvls(dA_mc, tp, rank, T, W, r, variant, d, z_own, s_own, dP_mc, dss_mc, ST(stream));
}

int btp_counter_add(int* ctr, int delta, void* stream) { return btp::counter_add(ctr, delta, ST(stream)); }

int btp_reduce_rows(const float* in, int splits, long long split_stride, long long ldi, int rows, int cols,
                    const float* col_scale, float* out, long long ldo, int accumulate, void* stream) {
  return btp::reduce_rows(in, splits, split_stride, ldi, rows, cols, col_scale, out, ldo, accumulate, ST(stream));
}

int btp_zero(void* ptr, long long bytes, void* stream) {
  if (bytes < 0) return BTP_ERR_DIM;
  if (bytes == 0) return BTP_OK;
  return cudaMemsetAsync(ptr, 0, (size_t)bytes, ST(stream)) == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int btp_num_sms(void) { return btp::num_sms_cached(); }

const char* btp_version(void) { return "btp-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
