#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/btp.h"

namespace btp {
int num_sms_cached();
int gemm_launch(const btp_gemm_problem* probs, int n, int bn_hint, int max_ctas, cudaStream_t stream);
// scatter epilogue: each problem's output rows are reduce-added into the owning rank's buffer
struct ScatterSpec {
  int n_owners;             // tp
  void* const* owners;      // host array: each owner's bf16 [rows_per_owner, width] buffer (ld)
  int rows_per_owner;       // T / tp, multiple of 32
  int width;                // columns of the owners' buffers
  long long ld;
  const int* col0;          // host array: first owner column of each problem
};
int gemm_launch_scatter(const btp_gemm_problem* probs, int n, int bn_hint, int max_ctas, cudaStream_t stream,
                        const ScatterSpec* sc);
int gemm_f32_launch(const btp_gemm_problem* probs, int n, cudaStream_t stream);
// f32 = false: bf16 activations (training path); true: fp32 activations (parity mode)
int rmsnorm_residual(const void* x, long long ldx, const void* branch, long long ldb, void* x_out, long long ldo,
                     const float* gamma, void* n_out, long long ldn, float* ss_out, float* rl_out, int rows,
                     int width, float eps, cudaStream_t st, bool f32);
int rmsnorm_apply(const void* x, long long ldx, const float* gamma, const float* ss_total, int d, float eps,
                  void* n_out, long long ldn, float* rms_out, int rows, int width, cudaStream_t st, bool f32);
int fixup_sigma_f32in(const float* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                      void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj, int variant,
                      cudaStream_t st);
int fixup_sigma(const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out, void* z_out,
                long long ldz, void* a_out, long long lda, int rows, int r, int nproj, int variant, cudaStream_t st,
                bool f32);
int fixup_sigma_bwd(const void* z, long long ldz, const void* da, long long ldda, const float* s, int d, void* dP,
                    long long lddp, float* dss, int rows, int r, int nproj, int variant, cudaStream_t st, bool f32);
int swiglu(const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda, int rows, int cols,
           cudaStream_t st, bool f32);
int swiglu_bwd(const void* g, long long ldg, const void* u, long long ldu, const void* dact, long long ldda,
               void* dg, long long lddg, void* du, long long lddu, int rows, int cols, cudaStream_t st, bool f32);
int rmsnorm_bwd(const void* dh, long long lddh, const void* x, long long ldx, const float* gamma, const float* dss,
                const void* dres, long long ldr, void* dx, long long lddx, float* dgamma_partial, int max_blocks,
                int* nblk_out, int rows, int width, cudaStream_t st, bool f32);
int rmsnorm_bwd_prep(const void* dn, long long lddn, const void* x, long long ldx, const float* gamma,
                     const float* s, void* dh, long long lddh, float* dss, int rows, int width, cudaStream_t st,
                     bool f32);
int reduce_rows(const float* in, int splits, long long split_stride, long long ldi, int rows, int cols,
                const float* col_scale, float* out, long long ldo, int accumulate, cudaStream_t st);
int add(const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows, int cols,
        cudaStream_t st, bool f32);
int dot(const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
        int max_blocks, int* nblk_out, cudaStream_t st, bool f32);
int adamw(float* master, float* m, float* v, const float* g, void* work, long long n, float lr, float b1, float b2,
          float eps, float wd, int step, const int* step_dev, cudaStream_t st, bool f32);
int counter_add(int* ctr, int delta, cudaStream_t st);
// model boundary (modelops.cu)
int embedding_fwd(const int* ids, const void* table, long long ldt, int vocab, int col0, void* out, long long ldo,
                  int rows, int width, int* bad, cudaStream_t st, bool f32);
int embedding_bwd(const int* ids, const void* dx, long long lddx, int vocab, float* dtable, long long ldg, int rows,
                  int width, cudaStream_t st, bool f32);
int cross_entropy(const void* logits, long long ldl, const int* targets, int vocab, float* loss_rows, void* dlogits,
                  long long ldd, int rows, float scale, cudaStream_t st, bool f32);
// peer-memory chunk boundaries (peer.cu)
int peer_signal(uint32_t* const* peer_flags, uint32_t* epoch, int slot, int rank, int tp, cudaStream_t st);
int peer_wait(const uint32_t* flags, const uint32_t* epoch, int slot, int tp, cudaStream_t st);
int peer_boundary_fwd(const void* const* P_peers, const float* const* ss_peers, int tp, int rank, int T, int W, int r,
                      int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                      cudaStream_t st, void* R_own = nullptr);
int peer_boundary_bwd(const void* const* da_peers, int tp, int rank, int T, int W, int r, int variant, int d,
                      const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                      cudaStream_t st, void* R_own = nullptr);
int peer_boundary_fwd_nvls(const void* P_mc, const float* ss_mc, int tp, int rank, int T, int W, int r, int variant,
                           int d, float eps, void* z_own, float* s_own, void* a_mc, cudaStream_t st);
int peer_boundary_bwd_nvls(const void* dA_mc, int tp, int rank, int T, int W, int r, int variant, int d,
                           const void* z_own, const float* s_own, void* dP_mc, float* dss_mc, cudaStream_t st);
// attention (attn.cu)
int attn_tune(int key, int value);
int attn_fwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, void* o,
             long long ldo, float* lse, int b, int s, int h, int hd, cudaStream_t stream, long long* trace = nullptr);
int attn_bwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, const void* o,
             long long ldo, const void* dO, long long lddo, const float* lse, float* D, float* dq_acc,
             long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv, long long lddv, int b,
             int s, int h, int hd, cudaStream_t stream, long long* trace = nullptr);
}  // namespace btp
