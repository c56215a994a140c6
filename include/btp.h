/*
 * btp.h — C-ABI of the B200-native Bottleneck-aware Tensor Parallelism (BTP) block step.
 *
 * Plain pointers and sizes only: every pointer is a DEVICE pointer owned by the caller
 * (kernels never allocate), every call is asynchronous on the caller's cudaStream_t
 * (passed as void*), and every entry point returns a btp_status.
 *
 * The reference (`btpsim`, pure Python/NumPy) has no FFI; each entry point below replaces
 * one compute site of its executor. The replaced reference symbol is cited per function
 * (paths relative to the reference package root `pkg/src/btpsim/`).
 *
 * Precision: bf16 storage for activations and GEMM operands, fp32 accumulation (TMEM),
 * fp32 for every per-row statistic (sum of squares, local/global RMS), fp32 weight grads.
 */
#ifndef BTP_H_
#define BTP_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef enum btp_status {
  BTP_OK = 0,
  BTP_ERR_DIM = 1,          /* shapes do not conform (reference DimensionError / PlanError) */
  BTP_ERR_DIVISIBILITY = 2, /* dimension not divisible as required (reference DivisibilityError) */
  BTP_ERR_ALIGNMENT = 3,    /* TMA/vector alignment violated (row stride or width not a multiple of 8) */
  BTP_ERR_CUDA = 4          /* CUDA launch/runtime failure */
} btp_status;

/* One GEMM problem  C[M,N] = alpha * rowscale[m] * colscale[n] * sum_k A[m,k] B[n,k]  (+ resid[m,n]).
 *   A: a_mn == 0 -> row-major [M, K] (ld = lda);  a_mn == 1 -> row-major [K, M] (A transposed in memory)
 *   B: b_mn == 0 -> row-major [N, K] (ld = ldb);  b_mn == 1 -> row-major [K, N]
 *   C: bf16 (c_fp32 == 0) or fp32 (c_fp32 == 1) row-major [M, N] with ld = ldc.
 *   splits > 1: split-K; split s writes fp32 partial C + s*split_stride (reduce with btp_reduce_rows).
 * Replaces: tensor.py:71-83 `mm_values` (every GEMM), simulator.py:198-205 `_gemm_ranks`. */
typedef struct btp_gemm_problem {
  const void* a;
  long long lda;
  int a_mn;
  const void* b;
  long long ldb;
  int b_mn;
  void* c;
  long long ldc;
  int c_fp32;
  int M, N, K;
  const float* row_scale; /* [M] or NULL */
  const float* col_scale; /* [N] or NULL */
  const void* resid;      /* bf16 [M, ld_resid] or NULL (bf16 output only) */
  long long ld_resid;
  int splits;
  long long split_stride;
  float alpha; /* 0 is read as 1 */
  /* reduce_add: the epilogue adds its (scaled) tile into C with the TMA reduce-add (fp32 add
   * performed in L2) instead of storing it. Required for splits > 1 (split-K over the T tokens of
   * a weight gradient): C must be fp32 and zero-initialised (btp_zero); summation order across
   * splits is not fixed (fp32 round-off only). split_stride is unused. */
  int reduce_add;
  /* epilogue: 0 = store (with the optional resid add above);
   *           1 = rank-r boundary with sigma fused (TP = 1, where no all-reduce separates the
   *               down-projection from the activation): z = scale * acc -> C (bf16),
   *               a = crossgate(z) -> c2 (bf16), pairs (j, j + sigma_half) within each
   *               2*sigma_half-wide projection ([silu(u)*v, silu(v)*u], computed from bf16(z)).
   *               B must be K-major, N % (2*sigma_half) == 0, sigma_half % 64 == 0; no resid,
   *               split-K or reduce-add; every problem of the launch must use it.
   *               Replaces btp_fixup_sigma after the GEMM (model.py:189-196).
   *           2 = SwiGLU backward: acc = dact, resid = g (bf16), aux2 = u (bf16),
   *               C = dg = dact*u*silu'(g), c2 = du = dact*silu(g)   (both bf16, no split-K)
   * Aux inputs are TMA-loaded into the epilogue's swizzled staging buffers, prefetched one
   * chunk ahead; outputs leave through TMA bulk stores. */
  int epilogue;
  const void* aux2;
  long long ld_aux2;
  void* c2;
  long long ldc2;
  int sigma_half; /* epilogue 1: r/2 (half-width of the crossgate pairs) */
} btp_gemm_problem;

/* Grouped/batched tcgen05 GEMM: n (1..8) independent problems in ONE persistent launch.
 * All problems share (a_mn, b_mn). bn_hint: 0 = auto, 128 or 256 = N tile.
 * Replaces: simulator.py:208-218 `_gemm_ranks_batched`, tensor.py:97-112 `batched_matmul`
 * (grouped up-projections q|k|v and gate|up, simulator.py:655-668). */
int btp_gemm(const btp_gemm_problem* problems, int n, int bn_hint, void* stream);

/* btp_gemm with the reduce-scatter of a BTP chunk boundary fused into the epilogue (SURVEY §8f
 * row 2; replaces the row-parallel GEMM + the reduce half of SimGroup.all_reduce, simulator.py:
 * 605-616): output rows [o * rows_per_owner, (o + 1) * rows_per_owner) of every problem are
 * TMA reduce-added in 32 x 32 fp32 chunks (the add performed at the destination) into owners[o] —
 * rank o's fp32 [rows_per_owner, width] buffer (row stride ld, rows_per_owner % 32 == 0),
 * normally peer-mapped memory of another GPU — at columns col0[p] + n, as the tiles finish,
 * instead of being stored. Plain epilogue only (row /
 * column scale allowed; no residual, split-K or fp32 output); problem c pointers may be NULL.
 * The owners' buffers must hold zeros (or the partial sums of other ranks) before the launch;
 * the reduced values are complete once every rank's launch has finished (signal with
 * btp_peer_signal on the same stream). owners / col0 are HOST arrays (n_owners / n entries). */
int btp_gemm_scatter(const btp_gemm_problem* problems, int n, int bn_hint, void* const* owners, int n_owners,
                     int rows_per_owner, int width, long long ld, const int* col0, void* stream);

/* Tile mode switch for btp_gemm: 1 = CTA-pair tiles (cluster of 2 CTAs on one TPC,
 * tcgen05.mma.cta_group::2, 256 x BN per pair) for launches with plain / sigma epilogues
 * (residual epilogues stay single-CTA); 2 (default) = pair tiles for residual epilogues too;
 * 0 = single-CTA 128 x BN tiles everywhere. Returns the previous setting. */
int btp_gemm_set_pair(int enable);
/* Residual epilogues: 3 (default) by output width — every residual problem N <= 1024 (the TP >= 2
 * o / down up-projections): pipelined residual slots refilled one tile ahead by a producer warp,
 * with st.global stores; wider: stage a tile's whole residual. 2 = always the pipeline (CTA-pair
 * launches), 1 = always whole-tile staging (four 64-column chunk buffers per epilogue warp, one TMA
 * round trip per tile), 0 = per-chunk prefetch. Returns the previous value. */
int btp_gemm_set_res4(int enable);
/* Epilogue stores: 0 (default) TMA bulk-tensor stores, 1 = coalesced st.global from the swizzled
 * staging chunk (4 rows x 128 B per warp instruction) for every launch. Split-K reduce-adds and the
 * scatter mode always use the TMA reduce. Returns the previous value. */
int btp_gemm_set_st_global(int enable);

/* Online RMSNorm (local form) fused with the residual add, one row per warp.
 *   v = x (+ branch); if x_out: x_out = bf16(v); stats use the rounded v
 *   ss[t] = sum_k v^2 ; rms_loc[t] = sqrt(ss/width + eps) ; n = v * gamma / rms_loc
 * n_out may be NULL (stat-only pass of the sync form). width <= 8192, width % 8 == 0.
 * Replaces: simulator.py:574-590 `norm_local` (online branch), norms.py:38-44 `local_sumsq`/
 * `local_rms`, residual adds simulator.py:687 / :706, norms.py:33-35 `rmsnorm_values` (width = d). */
int btp_rmsnorm_residual(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                         long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                         float* rms_loc_out, int rows, int width, float eps, void* stream);

/* Sync-form RMSNorm apply: n = x * gamma / sqrt(ss_total/d + eps); rms_out[t] = that sqrt.
 * Replaces: simulator.py:585-590 (sync branch of `norm_local`), norms.py:47-64 `sync_rmsnorm`. */
int btp_rmsnorm_apply(const void* x, long long ldx, const float* gamma, const float* ss_total, int d,
                      float eps, void* n_out, long long ldn, float* rms_out, int rows, int width,
                      void* stream);

/* Post-all-reduce fix-up and rank-r activation for one chunk boundary.
 *   if ss_total: s = sqrt(ss_total/d + eps) (written to s_out if non-NULL), z = P / s
 *   else       : z = P
 *   z_out = bf16(z) (skipped if z_out == P and no division);  a_out = sigma(z_out)
 *   sigma: variant 0 (svd) identity (a_out may be NULL); variant 1 (cola) crossgate per projection:
 *          [silu(u)*v, silu(v)*u] with u = z[:, p*r : p*r + r/2], v = z[:, p*r + r/2 : (p+1)*r]
 * Replaces: simulator.py:599-602 `correct`, :636 `/ rms_g`, :247-265 `_variant_a_input`,
 * model.py:189-196 `lowrank_crossgate_values`. */
int btp_fixup_sigma(const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                    void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj,
                    int variant, void* stream);

/* SwiGLU forward act = silu(g) * u.  Replaces tensor.py:131-132 `swiglu_values` (simulator.py:699). */
int btp_swiglu(const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda,
               int rows, int cols, void* stream);

/* SwiGLU backward: dg = dact * u * silu'(g), du = dact * silu(g). */
int btp_swiglu_bwd(const void* g, long long ldg, const void* u, long long ldu, const void* dact,
                   long long ldda, void* dg, long long lddg, void* du, long long lddu, int rows, int cols,
                   void* stream);

/* btp_fixup_sigma for an fp32 reduced partial P (bf16 z / a outputs; z_out required): the chunk
 * boundary all-reduced in fp32 (`boundary_dtype="fp32"`), so the cross-rank sum is rounded to
 * bf16 once, here, instead of once per ring hop. Same arguments and errors as btp_fixup_sigma. */
int btp_fixup_sigma_f32in(const float* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                          void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj,
                          int variant, void* stream);

/* Backward of `btp_fixup_sigma` for one chunk (sigma-bwd + normalisation-bwd, no collective):
 *   dz = sigma'(z) . da       (crossgate-bwd for variant 1, identity for 0)
 *   if s: dP = dz / s ;  dss[t] = -<dz_t, z_t> / (2 s^2 d)      else dP = dz
 * dP may alias da. Replaces the (absent) backward of simulator.py:592-653. */
int btp_fixup_sigma_bwd(const void* z, long long ldz, const void* da, long long ldda, const float* s, int d,
                        void* dP, long long lddp, float* dss, int rows, int r, int nproj, int variant,
                        void* stream);

/* Online/sync RMSNorm backward, rank-local (needs no collective):
 *   dx = dres + dh * gamma + 2 * x * dss[t]          (bf16 out; dres may be NULL)
 *   dgamma_partial[blk, k] = sum_{t in blk} dh[t,k] * x[t,k]   (fp32, nblk partial rows)
 * nblk partial rows are reduced by btp_reduce_rows. Returns the number of blocks used via *nblk. */
int btp_rmsnorm_bwd(const void* dh, long long lddh, const void* x, long long ldx, const float* gamma,
                    const float* dss, const void* dres, long long ldr, void* dx, long long lddx,
                    float* dgamma_partial, int max_blocks, int* nblk, int rows, int width, void* stream);

/* Replicated (full-width) RMSNorm backward prologue for the naive-TP / full-rank baselines,
 * n = x*gamma/s with s = sqrt(mean(x^2)+eps) saved by the forward:
 *   dh = dn / s (dh may alias dn),  dss[t] = -<dn_t, gamma*x_t> / (2 s^3 width)
 * then btp_rmsnorm_bwd(dh, x, gamma, dss, ...) yields dx and dgamma.
 * Replaces the (absent) backward of norms.py:27-35 `rmsnorm_reference`. */
int btp_rmsnorm_bwd_prep(const void* dn, long long lddn, const void* x, long long ldx, const float* gamma,
                         const float* s, void* dh, long long lddh, float* dss, int rows, int width, void* stream);

/* out[r, c] = (accumulate ? out : 0) + colscale[c] * sum_{s<splits} in[s*split_stride + r*ldi + c]
 * Deterministic (ascending split order) split-K / partial-sum reduction, fp32. */
int btp_reduce_rows(const float* in, int splits, long long split_stride, long long ldi, int rows, int cols,
                    const float* col_scale, float* out, long long ldo, int accumulate, void* stream);

/* out = a + b (bf16, elementwise over rows x cols). Replicated residual adds of the baselines
 * (simulator.py:367, :395, :523, :540), and the lax merge a = z + h_prev of the reduced rank-r
 * projection with the previous layer's bundle (simulator.py:260-265). */
int btp_add(const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows,
            int cols, void* stream);

/* partial[blk] = sum over a block's share of rows of <a_row, b_row> (bf16 in, fp32 out), for the
 * builder-defined loss L = sum(y * G) (the reference has no loss). Reduce the *nblk partials with
 * btp_reduce_rows; deterministic. */
int btp_dot(const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
            int max_blocks, int* nblk, void* stream);

/* ---- fp32 parity mode ------------------------------------------------------------------
 * The north_star's fp32 tolerance (1e-4 relative) cannot be met with single-pass TF32, so the
 * fp32 mode runs exact-fp32 CUDA kernels: a SIMT FFMA GEMM over the same problem descriptor
 * (A/B/C/resid fp32; epilogue 0 only; split-K computed in one pass, reduce_add honoured) and
 * fp32-activation twins of every row kernel (same arguments, T = float instead of bf16). */
int btp_gemm_f32(const btp_gemm_problem* problems, int n, void* stream);
int btp_rmsnorm_residual_f32(const void* x, long long ldx, const void* branch, long long ldb, void* x_out,
                             long long ldo, const float* gamma, void* n_out, long long ldn, float* ss_out,
                             float* rms_loc_out, int rows, int width, float eps, void* stream);
int btp_rmsnorm_apply_f32(const void* x, long long ldx, const float* gamma, const float* ss_total, int d,
                          float eps, void* n_out, long long ldn, float* rms_out, int rows, int width, void* stream);
int btp_fixup_sigma_f32(const void* P, long long ldp, const float* ss_total, int d, float eps, float* s_out,
                        void* z_out, long long ldz, void* a_out, long long lda, int rows, int r, int nproj,
                        int variant, void* stream);
int btp_swiglu_f32(const void* g, long long ldg, const void* u, long long ldu, void* act, long long lda, int rows,
                   int cols, void* stream);
int btp_swiglu_bwd_f32(const void* g, long long ldg, const void* u, long long ldu, const void* dact,
                       long long ldda, void* dg, long long lddg, void* du, long long lddu, int rows, int cols,
                       void* stream);
int btp_fixup_sigma_bwd_f32(const void* z, long long ldz, const void* da, long long ldda, const float* s, int d,
                            void* dP, long long lddp, float* dss, int rows, int r, int nproj, int variant,
                            void* stream);
int btp_rmsnorm_bwd_f32(const void* dh, long long lddh, const void* x, long long ldx, const float* gamma,
                        const float* dss, const void* dres, long long ldr, void* dx, long long lddx,
                        float* dgamma_partial, int max_blocks, int* nblk, int rows, int width, void* stream);
int btp_rmsnorm_bwd_prep_f32(const void* dn, long long lddn, const void* x, long long ldx, const float* gamma,
                             const float* s, void* dh, long long lddh, float* dss, int rows, int width,
                             void* stream);
int btp_add_f32(const void* a, long long lda, const void* b, long long ldb, void* out, long long ldo, int rows,
                int cols, void* stream);
int btp_dot_f32(const void* a, long long lda, const void* b, long long ldb, int rows, int cols, float* partial,
                int max_blocks, int* nblk, void* stream);

/* Fused AdamW over a flat parameter set of n elements (n % 8 == 0): fp32 master weights, fp32
 * first/second moments and fp32 gradients are updated in one pass and the working copy the
 * GEMMs read (bf16 for btp_adamw, fp32 for btp_adamw_f32) is rewritten from the master:
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr * ( (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps) + wd * p )
 * step is read from *step_dev when non-NULL (so a replayed CUDA graph keeps advancing it; bump it
 * with btp_counter_add after the update), else from `step`.
 * (the optimizer step over the sharded low-rank factors; absent in the reference.) */
int btp_adamw(float* master, float* m, float* v, const float* g, void* work, long long n, float lr, float b1,
              float b2, float eps, float wd, int step, const int* step_dev, void* stream);
int btp_adamw_f32(float* master, float* m, float* v, const float* g, void* work, long long n, float lr, float b1,
                  float b2, float eps, float wd, int step, const int* step_dev, void* stream);

/* ---- model boundary around the stack of BTP blocks (absent in the reference,
 * whose executor stops at the block and its tail all-gather, simulator.py:710-714; the paper
 * shards the embedding output so the first down-projection is row-split and replicates the
 * final projection). *_f32 twins take fp32 activations/tables.
 *
 * Embedding lookup of this rank's d-shard: out[t, :] = table[ids[t], col0 : col0 + width].
 * ids int32 [rows]; an id outside [0, vocab) yields a zero row and sets *bad = 1 (bad may be NULL). */
int btp_embedding_fwd(const int* ids, const void* table, long long ldt, int vocab, int col0, void* out,
                      long long ldo, int rows, int width, int* bad, void* stream);
int btp_embedding_fwd_f32(const int* ids, const void* table, long long ldt, int vocab, int col0, void* out,
                          long long ldo, int rows, int width, int* bad, void* stream);
/* Embedding backward: dtable[ids[t], :] += dx[t, :] (fp32, zero-initialised; fp32 atomics, so the
 * order in which repeated ids accumulate is not fixed). */
int btp_embedding_bwd(const int* ids, const void* dx, long long lddx, int vocab, float* dtable, long long ldg,
                      int rows, int width, void* stream);
int btp_embedding_bwd_f32(const int* ids, const void* dx, long long lddx, int vocab, float* dtable, long long ldg,
                          int rows, int width, void* stream);
/* Fused softmax cross-entropy over logits [rows, vocab] (vocab % 8 == 0), one pass for the
 * log-sum-exp and one for the gradient:
 *   loss_rows[t] = logsumexp(l_t) - l_t[target_t]                         (fp32)
 *   dlogits[t, j] = scale * (softmax(l_t)_j - [j == target_t])           (may alias logits; NULL = none)
 * target < 0 is the ignore index (loss 0, zero gradient). Reduce loss_rows with btp_reduce_rows. */
int btp_cross_entropy(const void* logits, long long ldl, const int* targets, int vocab, float* loss_rows,
                      void* dlogits, long long ldd, int rows, float scale, void* stream);
int btp_cross_entropy_f32(const void* logits, long long ldl, const int* targets, int vocab, float* loss_rows,
                          void* dlogits, long long ldd, int rows, float scale, void* stream);

/* ---- chunk boundaries over NVLink/NVSwitch peer memory ----------------
 * Replaces the SimGroup all-reduce (+ rider) at each BTP chunk boundary (simulator.py:153-181,
 * :592-653) AND the post-reduce fix-up + sigma (btp_fixup_sigma) with one kernel per chunk and
 * pass: reduce-scatter by pulling the rows this rank owns (T/tp consecutive rows, rank order sum
 * in fp32), fix-up + sigma on them, all-gather by pushing the results into every rank's buffer.
 * Every `*_peers` argument is a DEVICE array of tp pointers (rank order) into the symmetric
 * buffers of all ranks (peer-mapped memory); all bf16 row-major [T, W] with W = nproj * r.
 *
 * Flags: `flags` is this rank's symmetric uint32 array [nslots * tp]; `peer_flags` the device
 * array of every rank's flags pointer; `epoch` this rank's local uint32 [nslots] signal counters.
 * btp_peer_signal: after the stream's previous work, epoch[slot]++ and store it (release, system
 * scope) into flags_j[slot * tp + rank] of every rank j. btp_peer_wait: the stream waits until every
 * rank's flag for the slot has reached this rank's epoch[slot] (acquire, system scope). */
int btp_peer_signal(unsigned int* const* peer_flags, unsigned int* epoch, int slot, int rank, int tp, void* stream);
int btp_peer_wait(const unsigned int* flags, const unsigned int* epoch, int slot, int tp, void* stream);
/* Forward boundary: for owned rows t: P = sum_j P_j[t]; s = sqrt(sum_j ss_j[t]/d + eps) (ss_peers
 * NULL: s = 1); z_own[t - rank*T/tp] = bf16(P/s); s_own likewise (may be NULL); a = sigma(z)
 * (variant 1 crossgate over (j, j + r/2) pairs of each r-wide projection, 0 identity) stored into
 * a_j[t] of every rank. Call between a "ready" wait and a "done" signal. */
int btp_peer_boundary_fwd(const void* const* P_peers, const float* const* ss_peers, int tp, int rank, int T, int W,
                          int r, int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                          void* stream);
/* Backward boundary: for owned rows t: da = sum_j da_j[t]; dz = sigma'(z_own) da; dP = dz / s
 * (s_own NULL: s = 1) stored into dP_j[t] of every rank; with s_own: dss_j[t] = -<dz, z>/(2 s^2 d)
 * for every rank (dss_peers may be NULL). Replaces the backward all-reduce + btp_fixup_sigma_bwd. */
int btp_peer_boundary_bwd(const void* const* da_peers, int tp, int rank, int T, int W, int r, int variant, int d,
                          const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                          void* stream);

/* The boundary halves that follow btp_gemm_scatter: the partial sums of every rank have already been
 * reduce-added into this rank's owned rows R_own (fp32 [T/tp, W], local); the kernel reads them
 * (and re-zeroes them for the next use), then does the same fix-up / sigma / push (forward) or
 * sigma-bwd / push (backward) as btp_peer_boundary_fwd / _bwd. */
int btp_peer_boundary_fwd_local(void* R_own, const float* const* ss_peers, int tp, int rank, int T, int W, int r,
                                int variant, int d, float eps, void* z_own, float* s_own, void* const* a_peers,
                                void* stream);
int btp_peer_boundary_bwd_local(void* R_own, int tp, int rank, int T, int W, int r, int variant, int d,
                                const void* z_own, const float* s_own, void* const* dP_peers, float* const* dss_peers,
                                void* stream);

/* NVLS (NVLink SHARP) boundaries: *_mc are NVSwitch MULTICAST addresses of the symmetric buffers
 * (every rank's copy bound to one multicast object). Owned rows are read with multimem.ld_reduce
 * (the switch sums the tp partials, fp32 accumulation) and a / dP (and dss) are written once with
 * multimem.st (the switch replicates them to every rank): 2/tp of T·W·2 B per rank over NVLink
 * instead of 2(tp-1)/tp. Same math, flags and ordering as btp_peer_boundary_fwd / _bwd. */
int btp_peer_boundary_fwd_nvls(const void* P_mc, const float* ss_mc, int tp, int rank, int T, int W, int r,
                               int variant, int d, float eps, void* z_own, float* s_own, void* a_mc, void* stream);
int btp_peer_boundary_bwd_nvls(const void* dA_mc, int tp, int rank, int T, int W, int r, int variant, int d,
                               const void* z_own, const float* s_own, void* dP_mc, float* dss_mc, void* stream);

/* ---- attention (reference model.py:205-230 `sdpa_values`, simulator.py:221-233) ----------------
 * Unmasked softmax(q k^T / sqrt(hd)) v per (batch, head) on tcgen05 / TMEM. q, k, v, o are bf16
 * row-major [b*s, >= h*hd] with row strides ld* (elements, multiple of 8) and head j at columns
 * [j*hd, (j+1)*hd): the reference's heads-as-contiguous-feature-slices layout. s % 128 == 0,
 * hd in {64, 128}. lse (fp32 [b, h, s]) receives the log2-domain log-sum-exp of the scaled scores,
 * log2(sum_k exp2(q.k * log2(e)/sqrt(hd))), the statistics the backward recomputes P from. */
int btp_attn_fwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv, void* o,
                 long long ldo, float* lse, int b, int s, int h, int hd, void* stream);

/* Attention backward for btp_attn_fwd's output o and lse: dq, dk, dv (bf16, same layout as q/k/v)
 * from dO. Workspaces: D fp32 [b, h, s] (rowsum(dO o O)), dq_acc fp32 [b*s, >= h*hd] (row stride
 * ldacc, zeroed and summed over the key tiles inside the call). Three launches: the D / zero pass,
 * the tcgen05 kernel (one CTA per key tile walking every query tile; dK / dV in TMEM, dQ reduced
 * into dq_acc), the dq conversion. Replaces the reference's (absent) attention backward: the
 * analytic derivative of model.py:205-230. */
int btp_attn_bwd(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                 const void* o, long long ldo, const void* dO, long long lddo, const float* lse, float* D,
                 float* dq_acc, long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv,
                 long long lddv, int b, int s, int h, int hd, void* stream);

/* btp_attn_bwd with pipeline diagnostics: the CTA of key tile 0 / head 0 / batch 0 writes clock64()
 * stamps of its warp roles into trace (int64 [s/128, 16], device memory) per query tile. */
int btp_attn_bwd_trace(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                       const void* o, long long ldo, const void* dO, long long lddo, const float* lse, float* D,
                       float* dq_acc, long long ldacc, void* dq, long long lddq, void* dk, long long lddk, void* dv,
                       long long lddv, int b, int s, int h, int hd, long long* trace, void* stream);

/* btp_attn_fwd with pipeline diagnostics (split-row kernel): the CTA of query tile 0 / head 0 / batch 0
 * writes clock64() stamps of its warp roles into trace (int64 [s/128, 16], device memory) per key tile. */
int btp_attn_fwd_trace(const void* q, long long ldq, const void* k, long long ldk, const void* v, long long ldv,
                       void* o, long long ldo, float* lse, int b, int s, int h, int hd, long long* trace, void* stream);

/* Attention tuning knobs (host-side state read at launch; graph captures keep their choice). key 0: every
 * n-th exp2 pair of the forward softmax on the FMA pipe (polynomial) instead of the MUFU (n in {0 = none,
 * 2, 3, 4, 5}, default 2); key 1: forward kernel (4 = two query tiles per CTA sharing K / V, default when
 * s % 256 == 0; 3 = split rows, one S buffer, two CTAs per SM; 2 / 1 = split rows, double-buffered S, 4 / 2
 * key groups; 0 = single S buffer, two CTAs per SM; hd 64 and s % 256 == 0 only: 5 = two query tiles with P in
 * its own TMEM columns, 6 = the same with each row split over two warps); key 2: in the hd-64 backward's P phase, every n-th group of four exp2s has two
 * on the FMA pipe (n in {0 = none, 1, 2 = default, 4}); key 3: hd-64 backward kernel (0 = the same 8 warps for P
 * and dS, default; 1 = split roles: P warps, alternating dS warp groups, dQ-reduce warps); keys 4 / 5:
 * diagnostics of the split-role kernel (WRONG results; 4: handshakes only, 5: bit 0 no dS stores, bit 1
 * no proxy fence, bit 2 no lse / D loads); key 6: forward diagnostics (split-row variants, WRONG results:
 * softmax warps only do the handshakes); key 7: hd-64 backward grid (1 = persistent, one CTA per SM walking
 * the key-tile work items, default; 0 = one CTA per key tile). value < 0 only queries. Returns the previous
 * value (-1: unknown key). */
int btp_attn_tune(int key, int value);

/* *ctr += delta on the stream (device-side step counters). */
int btp_counter_add(int* ctr, int delta, void* stream);

/* Zero `bytes` bytes of device memory on the stream (split-K reduce-add targets). */
int btp_zero(void* ptr, long long bytes, void* stream);

/* Number of SMs the library sizes persistent grids for (device 0 of the current context). */
int btp_num_sms(void);

/* Library version string. */
const char* btp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BTP_H_ */
