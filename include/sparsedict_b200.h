/*
 * sparsedict-B200 — C ABI of the CUDA (sm_100a) hot path.
 *
 * Plain pointers and sizes only. Every data pointer is a DEVICE pointer unless
 * stated; `stream` is a cudaStream_t passed as void*. Every call is
 * stream-ordered, never throws, never allocates caller-visible memory
 * (callers pass workspaces sized by the *_bytes queries) and returns 0 on
 * success or a negative code; sdb_last_error() describes the last failure on
 * the calling thread.
 *
 * dtype: SDB_F32 ("fast": FP32 arithmetic, tcgen05 3xTF32 correlation GEMM)
 *        SDB_F64 ("exact": FP64, bitwise identical OMP to the reference's
 *                 Numba kernels)
 *
 * Device layouts:
 *   Y      N x ldy   signal-major (row i = signal i)         == F-order m x N
 *   D      P x K x m atom-major per shard                    == F-order m x K
 *   G      P x K x K
 *   alpha0 N x lda
 *   shard_off  P+1 int64 signal offsets (shards are contiguous row ranges)
 *   codes  idx N x cap int32 (selection order), val N x cap, counts int32,
 *          status int8 (0 OK, 2 SINGULAR, 3 STALLED), rnorm
 *
 * Each entry cites the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/sparsedict/).
 */
#ifndef SPARSEDICT_B200_H
#define SPARSEDICT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDB_F32 0
#define SDB_F64 1
/* sdb_mod_update only: FP32 signal rows with FP64 code values (certified FP32
 * mode; the rows' values are exact in FP64 and all arithmetic is FP64) */
#define SDB_F32X 2

#define SDB_OK 0
#define SDB_EINVAL (-22)
#define SDB_ENOMEM (-12)
#define SDB_ECUDA (-5)
#define SDB_ENODEV (-19)
#define SDB_ENOTSUP (-95)

int sdb_abi_version(void);
const char *sdb_last_error(void);
/* compute capability major*10+minor of the current device, or <0 */
int sdb_device_cc(void);

/* Host->device ingest (replaces np.asarray/np.asfortranarray + the finiteness
 * checks, sparse_coding.py:241-245,267): dst[i*ldd + t] = (T)src[t*s_row +
 * i*s_col] for an m x N f64 matrix already copied to the device; *bad is set
 * to 1 if any entry is non-finite. */
int sdb_ingest(int dtype, int64_t m, int64_t N, const double *src, int64_t s_row, int64_t s_col,
               void *dst, int64_t ldd, int32_t *bad, void *stream);

/* dst (dtype) = src (f64), n elements (dictionary working copy). */
int sdb_cast(int dtype, int64_t n, const double *src, void *dst, void *stream);

/* Gram matrix per shard: _kernels.gram_matrix (_kernels.py:23-35), called once
 * per omp_batch (sparse_coding.py:269). D64 is (P,K,m) f64, G is (P,K,K) dtype.
 * F64: bitwise identical to the reference. */
int sdb_gram(int dtype, int64_t P, int64_t m, int64_t K, const double *D64, void *G, void *stream);

/* The same Gram matrix in both precisions from one pass (certified FP32 mode:
 * the coding kernels read G32, the certification G64): G32 = (float)G64, bitwise
 * what sdb_gram(SDB_F32) returns. */
int sdb_gram_pair(int64_t P, int64_t m, int64_t K, const double *D64, double *G64, float *G32, void *stream);

/* alpha0[i, j] = <d_j, y_i> with d from the shard of i: the c0 = D^T y loop of
 * omp_single (_kernels.py:54-59) for every signal at once. F64: bitwise
 * identical sequential sums. F32: tcgen05 3xTF32 GEMM when use_tc != 0 and the
 * shape is supported, FP32 SIMT otherwise. max_shard_rows = max shard size.
 * ws: sdb_correlate_workspace_bytes() (pre-split D_hi/D_lo for 3xTF32). */
int64_t sdb_correlate_workspace_bytes(int dtype, int64_t P, int64_t m, int64_t K);
int sdb_correlate(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off,
                  int64_t max_shard_rows, const void *Y, int64_t ldy, const void *D, void *alpha0,
                  int64_t lda, int use_tc, void *ws, int64_t ws_bytes, void *stream);

/* Batch OMP: _kernels.omp_batch_range (_kernels.py:161-173) over all N
 * signals, i.e. omp_single (:38-158) per signal: greedy selection with the
 * 1e-12 tie window and lowest-index tie-break, progressive Cholesky with the
 * singular guard `guard` (reference 1e-12), explicit residual, stop at
 * rnorm <= eps or cap atoms. Fixed sparsity: cap = s, eps = 0. K <= 1024.
 * rnorm: optional output (NULL: residual norms not reported).
 * ysq: optional FP32 ||y_i||^2 from sdb_signal_sq (SDB_F32 only; NULL: formed
 * in the kernel). gap: optional FP32 output (SDB_F32 only; NULL: not reported):
 * the signal's smallest decision margin relative to ||y|| (best minus runner-up
 * |corr| above the rounding floor; | ||r|| - eps | at the explicit stopping
 * tests) -- the near-tie log sdb_certify re-decides in FP64.
 * scratch: sdb_omp_scratch_bytes() bytes; its first 256 bytes carry the FP32
 * kernel's work counter (signals are claimed in 32-signal chunks), the rest any per-warp
 * global scratch the generic kernel needs (NULL: static signal ranges). */
int64_t sdb_omp_scratch_bytes(int dtype, int64_t N, int64_t m, int64_t cap);
int sdb_omp(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off,
            const void *alpha0, int64_t lda, const void *Y, int64_t ldy, const void *D,
            const void *G, int64_t cap, double eps, double guard, int32_t *idx, void *val,
            int32_t *counts, int8_t *status, void *rnorm, const float *ysq, float *gap, void *scratch,
            int64_t scratch_bytes, void *stream);
/* Fused tensor-core Batch-OMP, FP32 (replaces sdb_correlate + sdb_omp for
 * _kernels.omp_batch_range, _kernels.py:161-173, when m <= 64, K <= 512 and
 * cap <= 8): tiles of 128 signals of one shard; every greedy step's
 * correlations D^T r are one tcgen05 kind::tf32 MMA of the tile's residuals
 * against the shard's dictionary resident in shared memory; the argmax is
 * decided exactly by re-evaluating in FP32 every atom within the TF32 error
 * window of the maximum (lowest index on ties); stall, singular-guard and eps
 * rules of omp_single (_kernels.py:61-154). No alpha0 matrix is formed.
 * D: P x K x m fp32 atom-major; G: P x K x K fp32. rnorm, gap optional
 * (gap[i] = the signal's smallest decision margin relative to ||y||: best
 * minus runner-up |corr| over the non-negligible steps and, in eps mode,
 * | ||r|| - eps | at every stopping test -- the near-tie log that
 * sdb_certify re-decides in FP64). ws: sdb_omp_tc_workspace_bytes(). */
/* FP64 certification of FP32 codes (the certified FP32 mode; replaces the
 * FP32 kernels' rounding by the reference's FP64 results, _kernels.py:38-173):
 * signals with status != 0 or a decision margin gap[i] < tau (gap may be NULL:
 * status only) are re-coded from scratch by the exact FP64 kernel (bitwise the
 * reference's omp_single for the same D, G, y) and listed in list[0..*nlist);
 * every other signal keeps its support and gets FP64 least-squares
 * coefficients on it. Y: the FP32 signal rows the FP32 kernels coded; Y64
 * (optional): the authoritative FP64 rows (used instead of Y when the FP32
 * rows are a rounding of them); D: P x K x m f64; Dt (optional): its P x m x K
 * transpose (coalesced c0 for the re-coded signals); G: the FP64
 * Gram (sdb_gram). idx/counts/status in-out; val (N x cap f64), rnorm (f64,
 * optional) out. list: N int32; nlist: 1 int32 (device). */
int sdb_certify(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off, const float *Y,
                const double *Y64, int64_t ldy, const double *D, const double *Dt, const double *G, int64_t cap, double eps, double tau,
                int32_t *idx, double *val, int32_t *counts, int8_t *status, double *rnorm, const float *gap,
                int32_t *list, int32_t *nlist, void *stream);
int sdb_omp_tc_supported(int64_t m, int64_t K, int64_t cap);
int64_t sdb_omp_tc_workspace_bytes(int64_t P, int64_t m, int64_t K);
int sdb_omp_tc(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off, const float *Y,
               int64_t ldy, const float *D, const float *G, int64_t cap, double eps, double guard,
               int32_t *idx, float *val, int32_t *counts, int8_t *status, float *rnorm, float *gap,
               void *ws, int64_t ws_bytes, void *stream);
/* Error-bounded FP32 coding in two launches (replaces sdb_correlate +
 * sdb_omp for the training loop's ε-mode passes, configs 2-3):
 * sdb_code_step1 is the tcgen05 correlation GEMM whose epilogue also runs the
 * first iteration of omp_single (_kernels.py:61-154: ||y|| <= eps early exit,
 * argmax with lowest-index tie-break, stall and singular tests, the
 * one-atom Cholesky solve and the eps test) on each signal's accumulator row,
 * with the exact arithmetic of sdb_omp's FP32 kernel. Signals it settles get
 * idx/val/counts/status written; the others get their alpha0 row stored and
 * status -1; their number is the int32 at ws + ws_bytes - 256 (reset by the
 * launch). sdb_omp_deferred (same ws, which also holds its work counter)
 * then codes exactly the status -1 signals. The union is bitwise sdb_omp's output
 * (rnorm not produced). Needs K <= 256, m <= 256, cap <= 32, eps > 0 and ysq
 * (sdb_signal_sq); SDB_ENOTSUP otherwise (the caller uses sdb_correlate +
 * sdb_omp). gap: optional FP32 decision margins of the settled signals (as
 * sdb_omp's; the deferred ones get theirs from sdb_omp_deferred), for
 * sdb_certify. ws: sdb_code_step1_workspace_bytes(). */
int64_t sdb_code_step1_workspace_bytes(int64_t P, int64_t m, int64_t K);
int sdb_code_step1(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off, const float *Y,
                   int64_t ldy, const float *D, const float *G, const float *ysq, int64_t cap, double eps,
                   double guard, float *alpha0, int64_t lda, int32_t *idx, float *val, int32_t *counts,
                   int8_t *status, float *gap, void *ws, int64_t ws_bytes, void *stream);
int sdb_omp_deferred(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off,
                     const float *alpha0, int64_t lda, const float *Y, int64_t ldy, const float *D,
                     const float *G, const float *ysq, int64_t cap, double eps, double guard, int32_t *idx,
                     float *val, int32_t *counts, int8_t *status, float *gap, void *ws, int64_t ws_bytes, void *stream);
/* ||y_i||^2 per signal (FP32, N floats) with the exact arithmetic of the
 * FP32 OMP kernel: passing it as sdb_omp's ysq gives bitwise the same codes
 * and lets the kernel skip loading y except near the eps threshold. */
int sdb_signal_sq(int64_t N, int64_t m, const float *Y, int64_t ldy, float *out, void *stream);

/* CSC packing (sparse_coding.py:294-303), in two stream-ordered phases:
 * indptr (N+1 int64) from counts, then indices (int64, ascending per column)
 * and data (f64). The caller reads indptr[N] (= nnz) to size the outputs. */
int64_t sdb_csc_workspace_bytes(int64_t N);
int sdb_csc_indptr(int64_t N, const int32_t *counts, int64_t *indptr, void *ws, void *stream);
int sdb_csc_fill(int dtype, int64_t N, int64_t cap, const int32_t *idx, const void *val,
                 const int32_t *counts, const int64_t *indptr, int64_t *indices, double *data,
                 void *stream);


/* MOD update for every shard at once: dictionary_update.mod_update
 * (dictionary_update.py:72-114). Codes are counting-sorted into per-atom
 * buckets (deterministic), A = X X^T and B = (Y X^T)^T are FP64 sequential
 * bucket sums, A Z = B is solved by a masked FP64 blocked Cholesky (unused
 * atoms -> identity rows, numerically dependent pivots -> atom dropped), then
 * residual_fro = ||Y - Z^T X||_F (before normalisation), dead atoms
 * (usage 0 or norm <= 1e-12 max(maxnorm,1)) restored from D_prev and every
 * column normalised. Shards with no nonzero code return D_prev unchanged.
 * Outputs: D_out (P,K,m) f64, scales (P,K) raw column norms, usage (P,K),
 * dead (P,K), resid_fro (P), rank (P), deficient (P, dependent pivots).
 * residual_fro uses the least-squares identity ||Y - Z^T X||^2 = ||Y||^2 -
 * ||L^-1 B||^2; ysq_shard (P, optional) supplies ||Y_p||^2 (constant across
 * training iterations, see sdb_shard_energy), NULL computes it. */
int64_t sdb_mod_workspace_bytes(int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap);
int sdb_mod_update(int dtype, int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap,
                   const int64_t *shard_off, const void *Y, int64_t ldy, const int32_t *idx,
                   const void *val, const int32_t *counts, const double *D_prev, double *D_out,
                   double *scales, int32_t *usage, int8_t *dead, double *resid_fro, int32_t *rank,
                   int32_t *deficient, double rank_rcond, const double *ysq_shard, void *ws,
                   int64_t ws_bytes, void *stream);

/* out[p] = ||Y_p||_F^2 per shard (FP64, fixed reduction order); tmp holds N doubles. */
int sdb_shard_energy(int dtype, int64_t P, int64_t N, int64_t m, const int64_t *shard_off,
                     const void *Y, int64_t ldy, double *tmp, double *out, void *stream);

/* replace_degenerate_atoms (dictionary_update.py:117-177) per shard, in place
 * on D (P,K,m) f64: degenerate = usage 0 | norm <= 1e-12 | higher index of a
 * twin pair |<dn_i,dn_j>| > 0.999 (pairs in row-major order, the lower index
 * kept unless itself degenerate); each target (ascending) takes the next data
 * column by descending ||y - D x|| (ties to the lower column), zero columns
 * skipped. flags (P,K): 0 kept, 1 replaced, 2 unreplaced. ntarget (P). */
int64_t sdb_replace_workspace_bytes(int64_t P, int64_t N, int64_t m, int64_t K);
int sdb_replace_degenerate(int dtype, int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap,
                           const int64_t *shard_off, const void *Y, int64_t ldy,
                           const int32_t *idx, const void *val, const int32_t *counts,
                           const int32_t *usage, double *D, int8_t *flags, int32_t *ntarget,
                           void *ws, int64_t ws_bytes, void *stream);

/* usage (P,K) int32 = atom histogram of the codes per shard
 * (SparseCodeMatrix.row_usage, sparse_coding.py:122-124). */
int sdb_code_usage(int64_t P, int64_t N, int64_t K, int64_t cap, const int64_t *shard_off,
                   const int32_t *idx, const int32_t *counts, int32_t *usage, void *stream);

/* rsq[i] = ||y_i - D_p x_i||^2 (FP64), ysq[i] = ||y_i||^2 (ysq may be NULL):
 * the residual of metrics.mse_db (metrics.py:30-44) and of
 * dictionary_update.py:103,159. */
int sdb_residual_sq(int dtype, int64_t N, int64_t m, int64_t K, int64_t cap, int64_t P,
                    const int64_t *shard_off, const void *Y, int64_t ldy, const int32_t *idx,
                    const void *val, const int32_t *counts, const double *D, double *rsq,
                    double *ysq, void *stream);

/* out[p] = sum (or sqrt of the sum) of v over shard p, fixed reduction order. */
int sdb_shard_sum(int64_t P, const int64_t *shard_off, const double *v, double *out, int do_sqrt,
                  void *stream);

/* out[i] = sum_t val[i,t]^2 (per-signal code energy; ||X_t||_F^2 after a
 * shard sum — the merge weights of trainer.py:250). */
int sdb_code_energy(int dtype, int64_t N, int64_t cap, const void *val, const int32_t *counts,
                    double *out, void *stream);

/* first-columns init (trainer.py:145-148): D[p][a] = y_{off[p]+a} / ||.||,
 * zero_flag[p*K+a] = 1 for zero columns (host fills them from the seeded RNG). */
int sdb_first_columns(int dtype, int64_t P, int64_t K, int64_t m, const int64_t *shard_off,
                      const void *Y, int64_t ldy, double *D, int32_t *zero_flag, void *stream);

/* merge dataset (trainer.py:248-256): out[r] = w[r / group] * D[r], rows of m. */
int sdb_scale_rows(int dtype, int64_t rows, int64_t group, int64_t m, const double *D,
                   const double *w, void *out, void *stream);

/* out[r] = in[perm[r]] (rows of m values): split_dataset's column gather
 * (trainer.py:220-223) into shard-contiguous order. */
/* out[r] = src[perm[r]] (f64 rows of length m <= 256, cast to dtype) and
 * *bad = 1 if any gathered value is non-finite: split_dataset's gather fused
 * with the input cast and check. src may be device memory or pinned,
 * device-mapped host memory (see sdb_host_mapped): the rows then cross PCIe
 * directly in permuted order. */
int sdb_ingest_gather(int dtype, int64_t rows, int64_t m, const double *src, int64_t ldi,
                      const int64_t *perm, void *out, int64_t ldo, int32_t *bad, void *stream);
/* The same with the source's first drows rows also available in device memory
 * (dsrc, same row stride): those are read from HBM, the rest over PCIe. Lets
 * train_split_merge move the head of a host batch while the split permutation
 * is still being formed on the host. */
int sdb_ingest_gather_split(int dtype, int64_t rows, int64_t m, const double *src, int64_t ldi,
                            const int64_t *perm, const double *dsrc, int64_t drows, void *out, int64_t ldo,
                            int32_t *bad, void *stream);
/* Stream-ordered copy between any two UVA addresses (cudaMemcpyDefault). */
int sdb_copy_async(void *dst, const void *src, int64_t bytes, void *stream);
/* Device address of a pinned, device-mapped host allocation (UVA: normally the
 * same address); SDB_EINVAL for pageable memory. */
int sdb_host_mapped(const void *host, void **dev);
int sdb_gather_rows(int dtype, int64_t rows, int64_t m, const void *in, int64_t ldi,
                    const int64_t *perm, void *out, int64_t ldo, void *stream);

/* SparseCodeMatrix (CSC, sparse_coding.py:76-96) -> code rows (idx N x cap,
 * val, counts) for the MOD / residual kernels. cap >= max column nnz. */
int sdb_csc_to_codes(int dtype, int64_t N, int64_t cap, const int64_t *indptr,
                     const int64_t *indices, const double *data, int32_t *idx, void *val,
                     int32_t *counts, void *stream);

/* normalize_columns (dictionary_update.py:56-69) on atom-major rows of m:
 * out = row / ||row|| (zero rows untouched), scales = norms (may be NULL). */
int sdb_normalize(int64_t rows, int64_t m, const double *in, double *out, double *scales,
                  void *stream);

/* On-device synthetic sparse-model signals (replaces the host generator
 * synthesis.py:56-79 gen_signals, with the additive N(0, sigma^2) noise of the
 * BASELINE configs): Y[i*ldy + c] = sum_t coef_it D[a_it*m + c] + sigma n_ic,
 * s distinct uniform atoms a_it, coef, n ~ N(0,1) from a counter-based
 * Philox4x32-10 stream keyed by seed (each signal a fixed function of
 * (seed, i)). D: K x m f64 atom-major (unit columns). sup_out: optional
 * N x s int32 supports (draw order). dtype: output precision. */
int sdb_synth_sparse(int dtype, int64_t N, int64_t m, int64_t K, int64_t s, const double *D, double sigma,
                     uint64_t seed, void *Y, int64_t ldy, int32_t *sup_out, void *stream);

/* extract_patches (denoising.py:118-135): img H x W f64 row-major -> patches
 * (R*C) x p^2 signal-major in dtype, R = (H-p)/s+1, C = (W-p)/s+1. */
int sdb_extract_patches(int dtype, const double *img, int64_t H, int64_t W, int64_t p, int64_t s,
                        void *out, void *stream);

/* denoise_image tail (denoising.py:236-239 + :138-163): overlap-average the
 * patch estimates D x_k (computed on the fly from the codes), clip to
 * [lo, hi]. D is (K, p^2) f64 atom-major. */
int sdb_reconstruct(int dtype, int64_t H, int64_t W, int64_t p, int64_t s, const double *D,
                    int64_t cap, const int32_t *idx, const void *val, const int32_t *counts,
                    double lo, double hi, double *out, void *stream);

/* reconstruct_from_patches (denoising.py:138-163) on explicit estimates
 * P ((R*C) x p^2, signal-major f64). */
int sdb_reconstruct_dense(int64_t H, int64_t W, int64_t p, int64_t s, const double *P, double *out,
                          void *stream);

/* HOST function (no GPU): numpy.random.default_rng(seed).permutation(n) of
 * trainer.split_indices (trainer.py:208-209), bitwise identical, given the
 * PCG64 state numpy derives from the seed (bit_generator.state: 128-bit state
 * and increment split in hi/lo words, has_uint32, uinteger). out: n int64. */
int sdb_pcg64_permutation(int64_t n, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                          uint64_t inc_lo, int has_uint32, uint32_t uinteger, int64_t *out);
/* The same permutation split between host and device (n >= 2, n - 1 < 2^32,
 * has_uint32 = 0): the host parses the PCG64 stream into the Fisher-Yates
 * swap targets (js: n - 1 uint32, step k swaps n-1-k and js[k]; host-only,
 * js may be pinned memory), and the device resolves the swaps in parallel,
 * exactly (perm: n int64 device, ws: sdb_permutation_workspace_bytes). */
int sdb_pcg64_swap_targets(int64_t n, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                           uint64_t inc_lo, uint32_t *js);
int64_t sdb_permutation_workspace_bytes(int64_t n);
int sdb_permutation_from_targets(int64_t n, const uint32_t *js, int64_t *perm, void *ws,
                                 int64_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEDICT_B200_H */
