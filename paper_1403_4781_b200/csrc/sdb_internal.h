// Internal (C++) launch interface shared by the .cu translation units.
// The public C-ABI lives in include/sparsedict_b200.h / sdb_capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace sdb {

template <typename T>
struct OmpArgs {
    int64_t N;
    int m, K, cap, P;
    T eps, guard;
    const int64_t* shard_off;  // P+1 signal offsets
    const T* alpha0;           // N x lda
    int64_t lda;
    const T* Y;                // N x ldy
    int64_t ldy;
    const T* D;                // P x K x m (atom-major)
    const T* G;                // P x K x K
    int32_t* idx;              // N x cap
    T* val;                    // N x cap
    int32_t* counts;
    int8_t* status;
    T* rnorm;                  // optional (nullptr: not requested)
    const float* ysq;          // optional precomputed ||y||^2 (fast FP32 path only)
    int deferred;              // fast FP32 path: code only the signals with status == -1
    int* work;                 //   ... claiming 32-signal chunks from this zeroed counter
    unsigned char* gscratch;   // optional per-warp scratch in global memory
    int64_t gscratch_warps;
    int64_t warp_bytes;
    // exact kernel, certification mode: code only the signals list[0..*nlist)
    // (global row indices, outputs at those rows), y read from the FP32 rows
    // Yf, alpha0 == nullptr: c0 = D^T y formed in-kernel (reference order)
    const int32_t* list;
    const int32_t* nlist;
    const float* Yf;
    const T* Dt;               // optional: P x m x K transposed dictionary (coalesced in-kernel c0)
    // FP32 fast kernel: optional per-signal smallest decision margin / ||y||
    // (best vs runner-up |corr| above the rounding floor; | ||r|| - eps | at
    // every stopping test) for the FP64 certification pass
    float* gap;
};

int gram_f64(const double* D, int P, int64_t m, int64_t K, double* G, cudaStream_t st);
// FP64 certification of FP32 codes (sdb_certify.cu)
int certify_refit(int64_t N, int m, int K, int cap, int P, const int64_t* off, const float* Y, const double* Y64,
                  int64_t ldy,
                  const double* D, const double* G, const int32_t* idx, const int32_t* counts,
                  const int8_t* status, const float* gap, float tau, double* val, double* rnorm, int32_t* list,
                  int32_t* nlist, bool short_supports, cudaStream_t st);
int64_t perm_ws_bytes(int64_t n);
int perm_from_targets(int64_t n, const uint32_t* js, int64_t* perm, void* ws, int64_t ws_bytes,
                      cudaStream_t st);
int signal_sq_f32(int64_t N, int m, const float* Y, int64_t ldy, float* out, cudaStream_t st);
int gram_f32(const double* D, int P, int64_t m, int64_t K, float* G, cudaStream_t st);
int gram_screen_f32(const float* D, int P, int64_t m, int64_t K, float* G, cudaStream_t st);
int gram_f64_f32(const double* D, int P, int64_t m, int64_t K, double* G64, float* G32, cudaStream_t st);
int correlate_simt_f64(const double* Y, int64_t ldy, const int64_t* off, int64_t max_rows, int P,
                       const double* D, int64_t m, int64_t K, double* alpha, int64_t lda,
                       cudaStream_t st);
int correlate_simt_f32(const float* Y, int64_t ldy, const int64_t* off, int64_t max_rows, int P,
                       const float* D, int64_t m, int64_t K, float* alpha, int64_t lda,
                       cudaStream_t st);
// tcgen05 3xTF32 correlation GEMM (sdb_tc_gemm.cu); returns cudaErrorNotSupported
// when the shape is outside the kernel's tiling.
int correlate_tc_f32(int64_t N, const float* Y, int64_t ldy, const int64_t* off, int64_t max_rows,
                     int P, const float* D, int64_t m, int64_t K, float* alpha, int64_t lda, void* ws,
                     int64_t ws_bytes, cudaStream_t st);
int64_t corr_tc_ws_bytes(int P, int64_t m, int64_t K);
// the same GEMM with the first greedy OMP step fused into its epilogue (K <=
// 256): settled signals get their codes, the rest their alpha0 row and
// status -1 (their number added to *n_deferred)
int code_step1_tc_f32(int64_t N, const float* Y, int64_t ldy, const int64_t* off, int P, const float* D,
                      int64_t m, int64_t K, float* alpha, int64_t lda, void* ws, int64_t ws_bytes,
                      const float* ysq, const float* G, float eps, float guard, int cap, int32_t* idx,
                      float* val, int32_t* counts, int8_t* status, float* gap, int* n_deferred, cudaStream_t st);

template <typename T>
int launch_omp(OmpArgs<T> a, cudaStream_t st);

// fused tensor-core Batch-OMP (sdb_omp_tc.cu): FP32, m <= 64, K <= 512, cap <= 8
bool omp_tc_supported(int64_t m, int64_t K, int64_t cap);
int64_t omp_tc_ws_bytes(int64_t P, int64_t m, int64_t K);
int omp_tc_f32(int64_t N, int m, int K, int P, const int64_t* off, const float* Y, int64_t ldy, const float* D,
               const float* G, int cap, float eps, float guard, int32_t* idx, float* val, int32_t* counts,
               int8_t* status, float* rnorm, float* gap, void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t omp_warp_bytes_f32(int cap, int m);
int64_t omp_warp_bytes_f64(int cap, int m);

int64_t scan_workspace_bytes(int64_t N);
int exclusive_scan_counts(const int32_t* counts, int64_t N, int64_t* indptr, int64_t* ws,
                          cudaStream_t st);
template <typename T>
int pack_csc(int64_t N, int cap, const int32_t* idx, const T* val, const int32_t* counts,
             const int64_t* indptr, int64_t* out_idx, double* out_val, cudaStream_t st);

int synth_sparse(int dtype_f64, int64_t N, int m, int K, int s, const double* D, double sigma, uint64_t seed,
                 void* Y, int64_t ldy, int32_t* sup_out, cudaStream_t st);

}  // namespace sdb
