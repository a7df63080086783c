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

#define SDB_OK 0
#define SDB_EINVAL (-22)
#define SDB_ENOMEM (-12)
#define SDB_ECUDA (-5)
#define SDB_ENODEV (-19)

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

/* alpha0[i, j] = <d_j, y_i> with d from the shard of i: the c0 = D^T y loop of
 * omp_single (_kernels.py:54-59) for every signal at once. F64: bitwise
 * identical sequential sums. F32: tcgen05 3xTF32 GEMM when use_tc != 0 and the
 * shape is supported, FP32 SIMT otherwise. max_shard_rows = max shard size. */
int sdb_correlate(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off,
                  int64_t max_shard_rows, const void *Y, int64_t ldy, const void *D, void *alpha0,
                  int64_t lda, int use_tc, void *stream);

/* Batch OMP: _kernels.omp_batch_range (_kernels.py:161-173) over all N
 * signals, i.e. omp_single (:38-158) per signal: greedy selection with the
 * 1e-12 tie window and lowest-index tie-break, progressive Cholesky with the
 * singular guard `guard` (reference 1e-12), explicit residual, stop at
 * rnorm <= eps or cap atoms. Fixed sparsity: cap = s, eps = 0. K <= 1024.
 * scratch: sdb_omp_scratch_bytes() bytes (may be 0 -> pass NULL). */
int64_t sdb_omp_scratch_bytes(int dtype, int64_t N, int64_t m, int64_t cap);
int sdb_omp(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t *shard_off,
            const void *alpha0, int64_t lda, const void *Y, int64_t ldy, const void *D,
            const void *G, int64_t cap, double eps, double guard, int32_t *idx, void *val,
            int32_t *counts, int8_t *status, void *rnorm, void *scratch, int64_t scratch_bytes,
            void *stream);

/* CSC packing (sparse_coding.py:294-303), in two stream-ordered phases:
 * indptr (N+1 int64) from counts, then indices (int64, ascending per column)
 * and data (f64). The caller reads indptr[N] (= nnz) to size the outputs. */
int64_t sdb_csc_workspace_bytes(int64_t N);
int sdb_csc_indptr(int64_t N, const int32_t *counts, int64_t *indptr, void *ws, void *stream);
int sdb_csc_fill(int dtype, int64_t N, int64_t cap, const int32_t *idx, const void *val,
                 const int32_t *counts, const int64_t *indptr, int64_t *indices, double *data,
                 void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEDICT_B200_H */
