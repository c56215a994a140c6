// extern "C" boundary of libbtp.so: argument marshalling only; every entry point forwards
// to the kernels in gemm.cu / rowops.cu on the caller's stream. See include/btp.h.
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

extern "C" {

int btp_gemm(const btp_gemm_problem* problems, int n, int bn_hint, void* stream) {
  return btp::gemm_launch(problems, n, bn_hint, 0, ST(stream));
}

int btp_rmsnorm_residual(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                         long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                         float* rms_loc_out, int rows, int width, float eps, void* stream) {
  return btp::rmsnorm_residual(x, ldx, branch, ldb, x_out, ldo, gamma, n_out, ldn, ss_out, rms_loc_out, rows, width,
                               eps, ST(stream));
}

int btp_rmsnorm_apply(const void* x, long long ldx, const float* gamma, const float* ss_total, int d, float eps,
                      void* n_out, long long ldn, float* rms_out, int rows, int width, void* stream) {
  return btp::rmsnorm_apply(x, ldx, gamma, ss_total, d, eps, n_out, ldn, rms_out, rows, width, ST(stream));
}

int btp_fixup_sigma(const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                    void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj,
                    int variant, void* stream) {
  return btp::fixup_sigma(P, ldp, ss_total, d, eps, s_out, z_out, ldz, a_out, lda, rows, r, nproj, variant,
                          ST(stream));
}

int btp_swiglu(const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda, int rows,
               int cols, void* stream) {
  return btp::swiglu(g, ldg, u, ldu, act, lda, rows, cols, ST(stream));
}

int btp_swiglu_bwd(const void* g, long long ldg, const void* u, long long ldu, const void* dact, long long ldda,
                   void* dg, long long lddg, void* du, long long lddu, int rows, int cols, void* stream) {
  return btp::swiglu_bwd(g, ldg, u, ldu, dact, ldda, dg, lddg, du, lddu, rows, cols, ST(stream));
}

int btp_fixup_sigma_bwd(const void* z, long long ldz, const void* da, long long ldda, const float* s, int d,
                        void* dP, long long lddp, float* dss, int rows, int r, int nproj, int variant,
                        void* stream) {
  return btp::fixup_sigma_bwd(z, ldz, da, ldda, s, d, dP, lddp, dss, rows, r, nproj, variant, ST(stream));
}

int btp_rmsnorm_bwd(const void* dh, long long lddh, const void* x, long long ldx, const float* gamma,
                    const float* dss, const void* dres, long long ldr, void* dx, long long lddx,
                    float* dgamma_partial, int max_blocks, int* nblk, int rows, int width, void* stream) {
  return btp::rmsnorm_bwd(dh, lddh, x, ldx, gamma, dss, dres, ldr, dx, lddx, dgamma_partial, max_blocks, nblk, rows,
                          width, ST(stream));
}

int btp_reduce_rows(const float* in, int splits, long long split_stride, long long ldi, int rows, int cols,
                    const float* col_scale, float* out, long long ldo, int accumulate, void* stream) {
  return btp::reduce_rows(in, splits, split_stride, ldi, rows, cols, col_scale, out, ldo, accumulate, ST(stream));
}

int btp_add(const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows,
            int cols, void* stream) {
  return btp::add(a, lda, b, ldb, out, ldo, rows, cols, ST(stream));
}

int btp_rmsnorm_bwd_prep(const void* dn, long long lddn, const void* x, long long ldx, const float* gamma,
                         const float* s, void* dh, long long lddh, float* dss, int rows, int width, void* stream) {
  return btp::rmsnorm_bwd_prep(dn, lddn, x, ldx, gamma, s, dh, lddh, dss, rows, width, ST(stream));
}

int btp_dot(const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
            int max_blocks, int* nblk, void* stream) {
  return btp::dot(a, lda, b, ldb, rows, cols, partial, max_blocks, nblk, ST(stream));
}

int btp_zero(void* ptr, long long bytes, void* stream) {
  if (bytes < 0) return BTP_ERR_DIM;
  if (bytes == 0) return BTP_OK;
  return cudaMemsetAsync(ptr, 0, (size_t)bytes, ST(stream)) == cudaSuccess ? BTP_OK : BTP_ERR_CUDA;
}

int btp_num_sms(void) { return btp::num_sms_cached(); }

const char* btp_version(void) { return "btp-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
