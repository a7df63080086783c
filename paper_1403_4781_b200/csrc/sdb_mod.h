// MOD / replacement launch interface (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sdb {

struct ModWs {
    int64_t* cf;
    int32_t* chunk_hist;
    int64_t* chunk_off;
    int64_t* wpart;  // per-warp chunk-range partial counts (P x 8 x K)
    int64_t* bucket_off;
    int64_t* scan_ws;
    int32_t* bent;  // bucket entries: flat code index i * cap + slot
    double* A;
    double* B;
    double* rsq;
    int64_t* nnz;
    double* fmax;    // MOD-finish partials per (shard, 8-atom block)
    int64_t* fnnz;
    int32_t* frank;
    int32_t* deficient;
    int8_t* depmask;
    void* chol;
    double* wsq;
    double* ysqp;
    int32_t* need;
    double* mn;      // minimum-norm fallback slots (sdb_minnorm.cu)
    unsigned char* end;
};

template <typename T>
struct ModArgs {
    int P, m, K, cap;
    int64_t N;
    const int64_t* off;
    const T* Y;
    const float* Yf;       // optional (T = double): FP32 rows whose values are the FP64 ones
    int64_t ldy;
    const int32_t* idx;
    const T* val;
    const int32_t* counts;
    const double* Dprev;   // P x K x m
    double* Dout;          // P x K x m
    double* scales;        // P x K
    int32_t* usage;        // P x K
    int8_t* dead;          // P x K
    double* resid_fro;     // P
    int32_t* rank;         // P
    int32_t* deficient_out;  // P (optional)
    int64_t* nnz_out;        // P (optional)
    double rank_rcond;
    const double* ysq_shard;  // optional (P): ||Y_p||_F^2, else computed
    void* ws;
};

template <typename T>
struct ReplaceArgs {
    int P, m, K, cap;
    int64_t N;
    const int64_t* off;
    const T* Y;
    int64_t ldy;
    const int32_t* idx;
    const T* val;
    const int32_t* counts;
    const int32_t* usage;
    double* D;             // in/out
    int8_t* flags;         // P x K: 0 kept, 1 replaced, 2 unreplaced
    int32_t* ntarget_out;  // P (optional)
    void* ws;
};

int64_t mod_ws_bytes(int P, int64_t N, int m, int K, int cap);
// pivot tolerance (relative to the largest used diagonal of X X^T) at which the
// Cholesky flags a shard for the minimum-norm (Jacobi pseudo-inverse) solve
constexpr double MN_FLAG_TOL = 1e-8;
int64_t minnorm_ws_bytes(int P, int m, int K);
template <typename TY, typename T>
int minnorm_solve(int P, int K, int m, const TY* Y, int64_t ldy, int cap, const int32_t* idx, const T* val,
                  const int32_t* counts, const int64_t* bucket_off, const int32_t* bent, const int32_t* usage,
                  double rcond, double* A, double* B, int32_t* deficient, double* wsq, double* slots,
                  cudaStream_t st);
template <typename T> int mod_update(const ModArgs<T>& a, cudaStream_t st);
int64_t replace_ws_bytes(int P, int64_t N, int m, int K);
template <typename T> int replace_degenerate(const ReplaceArgs<T>& a, cudaStream_t st);
template <typename T>
int residual_sq(int64_t N, int m, int K, int cap, int P, const int64_t* off, const T* Y, int64_t ldy,
                const int32_t* idx, const T* val, const int32_t* counts, const double* D,
                double* rsq, double* ysq, cudaStream_t st);
int shard_ysq(int P, int64_t N, int m, const void* Y, int64_t ldy, bool f64, const int64_t* off,
              double* tmp, double* out, cudaStream_t st);
int shard_sum(int P, const int64_t* off, const double* v, double* out, int do_sqrt, cudaStream_t st);
int usage_direct(int64_t N, int K, int cap, int P, const int64_t* off, const int32_t* idx,
                 const int32_t* counts, int32_t* usage, cudaStream_t st);
template <typename T>
int code_sq(int64_t N, int cap, const T* val, const int32_t* counts, double* out, cudaStream_t st);
template <typename T>
int first_columns(int P, int K, int m, const int64_t* off, const T* Y, int64_t ldy, double* D,
                  int32_t* zero_flag, cudaStream_t st);
template <typename T>
int scale_rows(int64_t rows, int group, int m, const double* D, const double* w, T* out, cudaStream_t st);

}  // namespace sdb
