// C-ABI entry points (include/sparsedict_b200.h). Validation of sizes and
// dtypes happens here; data-dependent preconditions (unit-norm dictionary,
// finite inputs, mode choice) are checked by the Python boundary before any
// launch, as the reference does (sparse_coding.py:145-155, 241-264).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>

#include "../../include/sparsedict_b200.h"
#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_mod.h"
#include "sdb_aux.h"

namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_rc(int rc, const char* where) {
    if (rc == 0) return SDB_OK;
    return fail(SDB_ECUDA, "%s: %s", where, cudaGetErrorString((cudaError_t)rc));
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }
inline bool dtype_ok(int dt) { return dt == SDB_F32 || dt == SDB_F64; }

template <typename T>
__global__ void k_ingest(int64_t m, int64_t N, const double* __restrict__ src, int64_t s_row,
                         int64_t s_col, T* __restrict__ dst, int64_t ldd, int32_t* bad) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * N) return;
    const int64_t i = e / m, t = e % m;
    const double v = src[t * s_row + i * s_col];
    if (!isfinite(v)) *bad = 1;
    dst[i * ldd + t] = (T)v;
}

template <typename T>
__global__ void k_cast(int64_t n, const double* __restrict__ src, T* __restrict__ dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) dst[e] = (T)src[e];
}
}  // namespace

extern "C" {

int sdb_abi_version(void) { return 12; }
const char* sdb_last_error(void) { return g_err.c_str(); }

int sdb_device_cc(void) {
    int dev = 0, ma = 0, mi = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(SDB_ENODEV, "no CUDA device");
    cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev);
    return ma * 10 + mi;
}

int sdb_ingest(int dtype, int64_t m, int64_t N, const double* src, int64_t s_row, int64_t s_col,
               void* dst, int64_t ldd, int32_t* bad, void* stream) {
    if (!dtype_ok(dtype) || m < 0 || N < 0 || ldd < m) return fail(SDB_EINVAL, "sdb_ingest: bad args");
    if (m * N == 0) return SDB_OK;
    const int64_t tot = m * N;
    const unsigned blocks = (unsigned)((tot + 255) / 256);
    if (dtype == SDB_F32)
        k_ingest<float><<<blocks, 256, 0, S(stream)>>>(m, N, src, s_row, s_col, (float*)dst, ldd, bad);
    else
        k_ingest<double><<<blocks, 256, 0, S(stream)>>>(m, N, src, s_row, s_col, (double*)dst, ldd, bad);
    return cuda_rc((int)cudaGetLastError(), "sdb_ingest");
}

int sdb_cast(int dtype, int64_t n, const double* src, void* dst, void* stream) {
    if (!dtype_ok(dtype) || n < 0) return fail(SDB_EINVAL, "sdb_cast: bad args");
    if (n == 0) return SDB_OK;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (dtype == SDB_F32)
        k_cast<float><<<blocks, 256, 0, S(stream)>>>(n, src, (float*)dst);
    else
        k_cast<double><<<blocks, 256, 0, S(stream)>>>(n, src, (double*)dst);
    return cuda_rc((int)cudaGetLastError(), "sdb_cast");
}

int sdb_gram(int dtype, int64_t P, int64_t m, int64_t K, const double* D64, void* G, void* stream) {
    if (!dtype_ok(dtype) || P < 1 || m < 1 || K < 1) return fail(SDB_EINVAL, "sdb_gram: bad args");
    int rc = dtype == SDB_F64 ? sdb::gram_f64(D64, (int)P, m, K, (double*)G, S(stream))
                              : sdb::gram_f32(D64, (int)P, m, K, (float*)G, S(stream));
    return cuda_rc(rc, "sdb_gram");
}

int sdb_gram_pair(int64_t P, int64_t m, int64_t K, const double* D64, double* G64, float* G32, void* stream) {
    if (P < 1 || m < 1 || K < 1 || G64 == nullptr || G32 == nullptr)
        return fail(SDB_EINVAL, "sdb_gram_pair: bad args");
    return cuda_rc(sdb::gram_f64_f32(D64, (int)P, m, K, G64, G32, S(stream)), "sdb_gram_pair");
}

int64_t sdb_correlate_workspace_bytes(int dtype, int64_t P, int64_t m, int64_t K) {
    return dtype == SDB_F32 ? sdb::corr_tc_ws_bytes((int)P, m, K) : 0;
}

int sdb_correlate(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off,
                  int64_t max_shard_rows, const void* Y, int64_t ldy, const void* D, void* alpha0,
                  int64_t lda, int use_tc, void* ws, int64_t ws_bytes, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || m < 1 || K < 1 || P < 1 || ldy < m || lda < K)
        return fail(SDB_EINVAL, "sdb_correlate: bad args");
    if (N == 0) return SDB_OK;
    int rc;
    if (dtype == SDB_F64) {
        rc = sdb::correlate_simt_f64((const double*)Y, ldy, shard_off, max_shard_rows, (int)P,
                                     (const double*)D, m, K, (double*)alpha0, lda, S(stream));
    } else {
        rc = cudaErrorNotSupported;
        if (use_tc)
            rc = sdb::correlate_tc_f32(N, (const float*)Y, ldy, shard_off, max_shard_rows, (int)P,
                                       (const float*)D, m, K, (float*)alpha0, lda, ws, ws_bytes,
                                       S(stream));
        if (rc == cudaErrorNotSupported)
            rc = sdb::correlate_simt_f32((const float*)Y, ldy, shard_off, max_shard_rows, (int)P,
                                         (const float*)D, m, K, (float*)alpha0, lda, S(stream));
    }
    return cuda_rc(rc, "sdb_correlate");
}

// scratch: [256 B: the FP32 kernel's work counter][per-warp global scratch
// when the generic kernel's state does not fit shared memory]
constexpr int64_t OMP_CTR_BYTES = 256;
// The dynamic chunk counter is a 32-bit int and every warp claims one chunk
// ahead, so it can overshoot N by up to 2 * warps * 32 (< 2^22): batches
// closer than that to 2^31 use static warp ranges / are rejected.
constexpr int64_t OMP_DYN_MAX_N = (int64_t(1) << 31) - (int64_t(1) << 22);

int64_t sdb_omp_scratch_bytes(int dtype, int64_t N, int64_t m, int64_t cap) {
    if (!dtype_ok(dtype) || cap < 1 || m < 1) return fail(SDB_EINVAL, "sdb_omp_scratch_bytes: bad args");
    const int64_t wb = dtype == SDB_F64 ? sdb::omp_warp_bytes_f64((int)cap, (int)m)
                                        : sdb::omp_warp_bytes_f32((int)cap, (int)m);
    if (wb * 8 <= 200 * 1024) return OMP_CTR_BYTES;  // the state fits shared memory
    const int64_t warps = std::max<int64_t>(8, std::min<int64_t>(((N + 7) / 8) * 8, (int64_t)148 * 32));
    return OMP_CTR_BYTES + wb * warps;
}

int sdb_omp(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off,
            const void* alpha0, int64_t lda, const void* Y, int64_t ldy, const void* D,
            const void* G, int64_t cap, double eps, double guard, int32_t* idx, void* val,
            int32_t* counts, int8_t* status, void* rnorm, const float* ysq, float* gap, void* scratch,
            int64_t scratch_bytes, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || lda < K)
        return fail(SDB_EINVAL, "sdb_omp: bad args");
    if (K > 1024) return fail(SDB_EINVAL, "sdb_omp: K=%lld > 1024 not supported", (long long)K);
    if (N == 0) return SDB_OK;
    const int64_t wb = dtype == SDB_F64 ? sdb::omp_warp_bytes_f64((int)cap, (int)m)
                                        : sdb::omp_warp_bytes_f32((int)cap, (int)m);
    const bool need_global = wb * 8 > 200 * 1024;
    if (need_global && (scratch == nullptr || scratch_bytes < OMP_CTR_BYTES + wb * 8))
        return fail(SDB_EINVAL, "sdb_omp: scratch of %lld bytes required", (long long)(OMP_CTR_BYTES + wb * 8));
    // a scratch of >= 256 bytes carries the FP32 kernel's chunk counter (zeroed here)
    int* work = (scratch != nullptr && scratch_bytes >= OMP_CTR_BYTES && N <= OMP_DYN_MAX_N) ? (int*)scratch
                                                                                            : nullptr;
    if (work) cudaMemsetAsync(work, 0, sizeof(int), S(stream));
    unsigned char* gscr = need_global ? (unsigned char*)scratch + OMP_CTR_BYTES : nullptr;
    const int64_t gscr_bytes = need_global ? scratch_bytes - OMP_CTR_BYTES : 0;
    auto fill = [&](auto& a) {
        a.N = N; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.P = (int)P;
        a.shard_off = shard_off; a.lda = lda; a.ldy = ldy;
        a.idx = idx; a.counts = counts; a.status = status;
        a.gscratch = gscr;
        a.gscratch_warps = need_global ? gscr_bytes / wb : 0;
        a.warp_bytes = wb;
    };
    int rc;
    if (dtype == SDB_F64) {
        sdb::OmpArgs<double> a{};
        fill(a);
        a.eps = eps; a.guard = guard;
        a.alpha0 = (const double*)alpha0; a.Y = (const double*)Y; a.D = (const double*)D;
        a.G = (const double*)G; a.val = (double*)val; a.rnorm = (double*)rnorm;
        rc = sdb::launch_omp<double>(a, S(stream));
    } else {
        sdb::OmpArgs<float> a{};
        fill(a);
        a.eps = (float)eps; a.guard = (float)guard;
        a.alpha0 = (const float*)alpha0; a.Y = (const float*)Y; a.D = (const float*)D;
        a.G = (const float*)G; a.val = (float*)val; a.rnorm = (float*)rnorm;
        a.ysq = ysq;
        a.work = work;
        a.gap = gap;
        rc = sdb::launch_omp<float>(a, S(stream));
    }
    return cuda_rc(rc, "sdb_omp");
}

// ---- fused tensor-core Batch-OMP (FP32): corr = D^T r per step on tcgen05
int sdb_certify(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off, const float* Y,
                const double* Y64, int64_t ldy, const double* D, const double* Dt, const double* G, int64_t cap, double eps, double tau, int32_t* idx, double* val,
                int32_t* counts, int8_t* status, double* rnorm, const float* gap, int32_t* list, int32_t* nlist,
                void* stream) {
    if (N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || !(tau >= 0.0) || list == nullptr ||
        nlist == nullptr)
        return fail(SDB_EINVAL, "sdb_certify: bad args");
    if (K > 1024 || m > 256 || cap > 32) return fail(SDB_ENOTSUP, "sdb_certify: needs K <= 1024, m <= 256, cap <= 32");
    if (N == 0) return SDB_OK;
    cudaMemsetAsync(nlist, 0, sizeof(int32_t), S(stream));
    int rc = sdb::certify_refit(N, (int)m, (int)K, (int)cap, (int)P, shard_off, Y, Y64, ldy, D, G, idx, counts, status,
                                gap, (float)tau, val, rnorm, list, nlist, eps > 0.0, S(stream));
    if (rc) return cuda_rc(rc, "sdb_certify (refit)");
    sdb::OmpArgs<double> a{};
    a.N = N; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.P = (int)P;
    a.shard_off = shard_off; a.lda = K; a.ldy = ldy;
    a.idx = idx; a.counts = counts; a.status = status;
    a.eps = eps; a.guard = 1e-12;              // the reference's guard (_kernels.py:18)
    a.alpha0 = nullptr; a.Y = Y64; a.Yf = Y64 ? nullptr : Y; a.D = D; a.G = G; a.val = val; a.rnorm = rnorm;
    a.list = list; a.nlist = nlist; a.Dt = Dt;
    a.warp_bytes = sdb::omp_warp_bytes_f64((int)cap, (int)m);
    return cuda_rc(sdb::launch_omp<double>(a, S(stream)), "sdb_certify (exact)");
}

int64_t sdb_omp_tc_workspace_bytes(int64_t P, int64_t m, int64_t K) {
    if (P < 1 || m < 1 || K < 1) return fail(SDB_EINVAL, "sdb_omp_tc_workspace_bytes: bad args");
    return sdb::omp_tc_ws_bytes(P, m, K);
}

int sdb_omp_tc_supported(int64_t m, int64_t K, int64_t cap) { return sdb::omp_tc_supported(m, K, cap) ? 1 : 0; }

int sdb_omp_tc(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off, const float* Y,
               int64_t ldy, const float* D, const float* G, int64_t cap, double eps, double guard,
               int32_t* idx, float* val, int32_t* counts, int8_t* status, float* rnorm, float* gap,
               void* ws, int64_t ws_bytes, void* stream) {
    if (N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || eps < 0.0)
        return fail(SDB_EINVAL, "sdb_omp_tc: bad args");
    if (!sdb::omp_tc_supported(m, K, cap))
        return fail(SDB_ENOTSUP, "sdb_omp_tc: needs m <= 64, K <= 512, cap <= 8");
    if (N > 0x7fffffffll) return fail(SDB_EINVAL, "sdb_omp_tc: N >= 2^31");
    if (N == 0) return SDB_OK;
    if (ws == nullptr || ws_bytes < sdb::omp_tc_ws_bytes(P, m, K))
        return fail(SDB_EINVAL, "sdb_omp_tc: workspace of %lld bytes required", (long long)sdb::omp_tc_ws_bytes(P, m, K));
    int rc = sdb::omp_tc_f32(N, (int)m, (int)K, (int)P, shard_off, Y, ldy, D, G, (int)cap, (float)eps,
                             (float)guard, idx, val, counts, status, rnorm, gap, ws, ws_bytes, S(stream));
    return cuda_rc(rc, "sdb_omp_tc");
}

// ---- fused first greedy step (error-bounded FP32 coding)
static int64_t step1_corr_bytes(int64_t P, int64_t m, int64_t K) {
    return (sdb::corr_tc_ws_bytes((int)P, m, K) + 255) / 256 * 256;
}

int64_t sdb_code_step1_workspace_bytes(int64_t P, int64_t m, int64_t K) {
    if (P < 1 || m < 1 || K < 1) return fail(SDB_EINVAL, "sdb_code_step1_workspace_bytes: bad args");
    return step1_corr_bytes(P, m, K) + 256;
}

int sdb_code_step1(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off, const float* Y,
                   int64_t ldy, const float* D, const float* G, const float* ysq, int64_t cap, double eps,
                   double guard, float* alpha0, int64_t lda, int32_t* idx, float* val, int32_t* counts,
                   int8_t* status, float* gap, void* ws, int64_t ws_bytes, void* stream) {
    if (N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || lda < K)
        return fail(SDB_EINVAL, "sdb_code_step1: bad args");
    if (K > 256 || m > 256 || cap > 32 || !(eps > 0.0) || ysq == nullptr)
        return fail(SDB_ENOTSUP, "sdb_code_step1: needs K <= 256, m <= 256, cap <= 32, eps > 0, ysq");
    if (ws == nullptr || ws_bytes < sdb_code_step1_workspace_bytes(P, m, K))
        return fail(SDB_EINVAL, "sdb_code_step1: workspace too small");
    if (N == 0) return SDB_OK;
    int32_t* counters = (int32_t*)((unsigned char*)ws + step1_corr_bytes(P, m, K));
    int rc = sdb::code_step1_tc_f32(N, Y, ldy, shard_off, (int)P, D, m, K, alpha0, lda, ws,
                                    step1_corr_bytes(P, m, K), ysq, G, (float)eps, (float)guard, (int)cap,
                                    idx, val, counts, status, gap, counters, S(stream));
    if (rc == cudaErrorNotSupported) return fail(SDB_ENOTSUP, "sdb_code_step1: shape outside the tcgen05 tiling");
    return cuda_rc(rc, "sdb_code_step1");
}

int sdb_omp_deferred(int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off,
                     const float* alpha0, int64_t lda, const float* Y, int64_t ldy, const float* D,
                     const float* G, const float* ysq, int64_t cap, double eps, double guard, int32_t* idx,
                     float* val, int32_t* counts, int8_t* status, float* gap, void* ws, int64_t ws_bytes,
                     void* stream) {
    if (N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || lda < K)
        return fail(SDB_EINVAL, "sdb_omp_deferred: bad args");
    if (K > 1024 || m > 256 || cap > 32 || ysq == nullptr)
        return fail(SDB_ENOTSUP, "sdb_omp_deferred: needs K <= 1024, m <= 256, cap <= 32 and ysq");
    if (ws == nullptr || ws_bytes < sdb_code_step1_workspace_bytes(P, m, K))
        return fail(SDB_EINVAL, "sdb_omp_deferred: the sdb_code_step1 workspace is required");
    if (N > OMP_DYN_MAX_N) return fail(SDB_ENOTSUP, "sdb_omp_deferred: N too close to 2^31 for the chunk counter");
    if (N == 0) return SDB_OK;
    sdb::OmpArgs<float> a{};
    a.N = N; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.P = (int)P;
    a.shard_off = shard_off; a.lda = lda; a.ldy = ldy;
    a.idx = idx; a.counts = counts; a.status = status;
    a.eps = (float)eps; a.guard = (float)guard;
    a.alpha0 = alpha0; a.Y = Y; a.D = D; a.G = G; a.val = val; a.rnorm = nullptr; a.ysq = ysq;
    a.deferred = 1;
    a.gap = gap;
    a.work = (int*)((unsigned char*)ws + step1_corr_bytes(P, m, K)) + 1;   // zeroed by sdb_code_step1
    return cuda_rc(sdb::launch_omp<float>(a, S(stream)), "sdb_omp_deferred");
}

int sdb_signal_sq(int64_t N, int64_t m, const float* Y, int64_t ldy, float* out, void* stream) {
    if (N < 0 || m < 1 || m > 256 || ldy < m || (N > 0 && (Y == nullptr || out == nullptr)))
        return fail(SDB_EINVAL, "sdb_signal_sq: bad args");
    return cuda_rc(sdb::signal_sq_f32(N, (int)m, Y, ldy, out, S(stream)), "sdb_signal_sq");
}

int64_t sdb_permutation_workspace_bytes(int64_t n) { return n < 1 ? 256 : sdb::perm_ws_bytes(n); }

int sdb_permutation_from_targets(int64_t n, const uint32_t* js, int64_t* perm, void* ws, int64_t ws_bytes,
                                 void* stream) {
    if (n < 1 || n - 1 > 0x7fffffffll || perm == nullptr || (n > 1 && (js == nullptr || ws == nullptr)))
        return fail(SDB_EINVAL, "sdb_permutation_from_targets: bad args");
    return cuda_rc(sdb::perm_from_targets(n, js, perm, ws, ws_bytes, S(stream)), "sdb_permutation_from_targets");
}

int64_t sdb_csc_workspace_bytes(int64_t N) { return sdb::scan_workspace_bytes(N < 1 ? 1 : N); }

int sdb_csc_indptr(int64_t N, const int32_t* counts, int64_t* indptr, void* ws, void* stream) {
    if (N < 0) return fail(SDB_EINVAL, "sdb_csc_indptr: bad args");
    int rc = sdb::exclusive_scan_counts(counts, N, indptr, (int64_t*)ws, S(stream));
    return cuda_rc(rc, "sdb_csc_indptr");
}

int sdb_csc_fill(int dtype, int64_t N, int64_t cap, const int32_t* idx, const void* val,
                 const int32_t* counts, const int64_t* indptr, int64_t* indices, double* data,
                 void* stream) {
    if (!dtype_ok(dtype) || N < 0 || cap < 1) return fail(SDB_EINVAL, "sdb_csc_fill: bad args");
    int rc = dtype == SDB_F64
                 ? sdb::pack_csc<double>(N, (int)cap, idx, (const double*)val, counts, indptr, indices, data, S(stream))
                 : sdb::pack_csc<float>(N, (int)cap, idx, (const float*)val, counts, indptr, indices, data, S(stream));
    return cuda_rc(rc, "sdb_csc_fill");
}


int64_t sdb_mod_workspace_bytes(int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap) {
    return sdb::mod_ws_bytes((int)P, N, (int)m, (int)K, (int)cap);
}

int sdb_mod_update(int dtype, int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap,
                   const int64_t* shard_off, const void* Y, int64_t ldy, const int32_t* idx,
                   const void* val, const int32_t* counts, const double* D_prev, double* D_out,
                   double* scales, int32_t* usage, int8_t* dead, double* resid_fro, int32_t* rank,
                   int32_t* deficient, double rank_rcond, const double* ysq_shard, void* ws,
                   int64_t ws_bytes, void* stream) {
    // dtype SDB_F32X: FP32 signal rows with FP64 code values (certified FP32
    // mode; the rows' values are exact, the arithmetic is FP64)
    if (!(dtype_ok(dtype) || dtype == SDB_F32X) || P < 1 || N < 0 || m < 1 || m > 256 || K < 1 || K > 1024 ||
        cap < 1 || ldy < m)
        return fail(SDB_EINVAL, "sdb_mod_update: bad args (m <= 256, K <= 1024)");
    if (N * cap > 0x7fffffffll)  // bucket entries are 32-bit flat code indices
        return fail(SDB_EINVAL, "sdb_mod_update: N * cap = %lld exceeds 2^31 - 1", (long long)(N * cap));
    if (ws == nullptr || ws_bytes < sdb::mod_ws_bytes((int)P, N, (int)m, (int)K, (int)cap))
        return fail(SDB_EINVAL, "sdb_mod_update: workspace too small");
    auto go = [&](auto* tag) {
        using T = std::remove_pointer_t<decltype(tag)>;
        sdb::ModArgs<T> a{};
        a.P = (int)P; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.N = N;
        a.off = shard_off; a.Y = (const T*)Y; a.ldy = ldy; a.idx = idx; a.val = (const T*)val;
        a.counts = counts; a.Dprev = D_prev; a.Dout = D_out; a.scales = scales; a.usage = usage;
        a.dead = dead; a.resid_fro = resid_fro; a.rank = rank; a.deficient_out = deficient;
        a.nnz_out = nullptr; a.rank_rcond = rank_rcond; a.ysq_shard = ysq_shard; a.ws = ws;
        if constexpr (std::is_same_v<T, double>) {
            if (dtype == SDB_F32X) { a.Y = nullptr; a.Yf = (const float*)Y; }
        }
        return sdb::mod_update<T>(a, S(stream));
    };
    int rc = (dtype == SDB_F64 || dtype == SDB_F32X) ? go((double*)nullptr) : go((float*)nullptr);
    return cuda_rc(rc, "sdb_mod_update");
}

int sdb_shard_energy(int dtype, int64_t P, int64_t N, int64_t m, const int64_t* shard_off,
                     const void* Y, int64_t ldy, double* tmp, double* out, void* stream) {
    if (!dtype_ok(dtype) || P < 1 || N < 0 || m < 1 || m > 256 || ldy < m)
        return fail(SDB_EINVAL, "sdb_shard_energy: bad args");
    return cuda_rc(sdb::shard_ysq((int)P, N, (int)m, Y, ldy, dtype == SDB_F64, shard_off, tmp, out,
                                  S(stream)), "sdb_shard_energy");
}

int64_t sdb_replace_workspace_bytes(int64_t P, int64_t N, int64_t m, int64_t K) {
    return sdb::replace_ws_bytes((int)P, N, (int)m, (int)K);
}

int sdb_replace_degenerate(int dtype, int64_t P, int64_t N, int64_t m, int64_t K, int64_t cap,
                           const int64_t* shard_off, const void* Y, int64_t ldy,
                           const int32_t* idx, const void* val, const int32_t* counts,
                           const int32_t* usage, double* D, int8_t* flags, int32_t* ntarget,
                           void* ws, int64_t ws_bytes, void* stream) {
    if (!dtype_ok(dtype) || P < 1 || N < 0 || m < 1 || m > 256 || K < 1 || cap < 1 || ldy < m)
        return fail(SDB_EINVAL, "sdb_replace_degenerate: bad args");
    if (ws == nullptr || ws_bytes < sdb::replace_ws_bytes((int)P, N, (int)m, (int)K))
        return fail(SDB_EINVAL, "sdb_replace_degenerate: workspace too small");
    auto go = [&](auto* tag) {
        using T = std::remove_pointer_t<decltype(tag)>;
        sdb::ReplaceArgs<T> a{};
        a.P = (int)P; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.N = N; a.off = shard_off;
        a.Y = (const T*)Y; a.ldy = ldy; a.idx = idx; a.val = (const T*)val; a.counts = counts;
        a.usage = usage; a.D = D; a.flags = flags; a.ntarget_out = ntarget; a.ws = ws;
        return sdb::replace_degenerate<T>(a, S(stream));
    };
    int rc = dtype == SDB_F64 ? go((double*)nullptr) : go((float*)nullptr);
    return cuda_rc(rc, "sdb_replace_degenerate");
}

int sdb_code_usage(int64_t P, int64_t N, int64_t K, int64_t cap, const int64_t* shard_off,
                   const int32_t* idx, const int32_t* counts, int32_t* usage, void* stream) {
    if (P < 1 || N < 0 || K < 1 || cap < 1) return fail(SDB_EINVAL, "sdb_code_usage: bad args");
    return cuda_rc(sdb::usage_direct(N, (int)K, (int)cap, (int)P, shard_off, idx, counts, usage,
                                     S(stream)), "sdb_code_usage");
}

int sdb_residual_sq(int dtype, int64_t N, int64_t m, int64_t K, int64_t cap, int64_t P,
                    const int64_t* shard_off, const void* Y, int64_t ldy, const int32_t* idx,
                    const void* val, const int32_t* counts, const double* D, double* rsq,
                    double* ysq, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || m < 1 || m > 256 || K < 1 || cap < 1 || P < 1 || ldy < m)
        return fail(SDB_EINVAL, "sdb_residual_sq: bad args");
    int rc = dtype == SDB_F64
                 ? sdb::residual_sq<double>(N, (int)m, (int)K, (int)cap, (int)P, shard_off, (const double*)Y,
                                            ldy, idx, (const double*)val, counts, D, rsq, ysq, S(stream))
                 : sdb::residual_sq<float>(N, (int)m, (int)K, (int)cap, (int)P, shard_off, (const float*)Y,
                                           ldy, idx, (const float*)val, counts, D, rsq, ysq, S(stream));
    return cuda_rc(rc, "sdb_residual_sq");
}

int sdb_shard_sum(int64_t P, const int64_t* shard_off, const double* v, double* out, int do_sqrt,
                  void* stream) {
    if (P < 1) return fail(SDB_EINVAL, "sdb_shard_sum: bad args");
    return cuda_rc(sdb::shard_sum((int)P, shard_off, v, out, do_sqrt, S(stream)), "sdb_shard_sum");
}

int sdb_code_energy(int dtype, int64_t N, int64_t cap, const void* val, const int32_t* counts,
                    double* out, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || cap < 1) return fail(SDB_EINVAL, "sdb_code_energy: bad args");
    int rc = dtype == SDB_F64 ? sdb::code_sq<double>(N, (int)cap, (const double*)val, counts, out, S(stream))
                              : sdb::code_sq<float>(N, (int)cap, (const float*)val, counts, out, S(stream));
    return cuda_rc(rc, "sdb_code_energy");
}

int sdb_first_columns(int dtype, int64_t P, int64_t K, int64_t m, const int64_t* shard_off,
                      const void* Y, int64_t ldy, double* D, int32_t* zero_flag, void* stream) {
    if (!dtype_ok(dtype) || P < 1 || K < 1 || m < 1 || ldy < m) return fail(SDB_EINVAL, "sdb_first_columns: bad args");
    int rc = dtype == SDB_F64
                 ? sdb::first_columns<double>((int)P, (int)K, (int)m, shard_off, (const double*)Y, ldy, D, zero_flag, S(stream))
                 : sdb::first_columns<float>((int)P, (int)K, (int)m, shard_off, (const float*)Y, ldy, D, zero_flag, S(stream));
    return cuda_rc(rc, "sdb_first_columns");
}

int sdb_scale_rows(int dtype, int64_t rows, int64_t group, int64_t m, const double* D,
                   const double* w, void* out, void* stream) {
    if (!dtype_ok(dtype) || rows < 0 || group < 1 || m < 1) return fail(SDB_EINVAL, "sdb_scale_rows: bad args");
    int rc = dtype == SDB_F64 ? sdb::scale_rows<double>(rows, (int)group, (int)m, D, w, (double*)out, S(stream))
                              : sdb::scale_rows<float>(rows, (int)group, (int)m, D, w, (float*)out, S(stream));
    return cuda_rc(rc, "sdb_scale_rows");
}


int sdb_gather_rows(int dtype, int64_t rows, int64_t m, const void* in, int64_t ldi,
                    const int64_t* perm, void* out, int64_t ldo, void* stream) {
    if (!dtype_ok(dtype) || rows < 0 || m < 1 || ldi < m || ldo < m) return fail(SDB_EINVAL, "sdb_gather_rows: bad args");
    int rc = dtype == SDB_F64 ? sdb::gather_rows<double>(rows, (int)m, (const double*)in, ldi, perm, (double*)out, ldo, S(stream))
                              : sdb::gather_rows<float>(rows, (int)m, (const float*)in, ldi, perm, (float*)out, ldo, S(stream));
    return cuda_rc(rc, "sdb_gather_rows");
}

int sdb_ingest_gather(int dtype, int64_t rows, int64_t m, const double* src, int64_t ldi, const int64_t* perm,
                      void* out, int64_t ldo, int32_t* bad, void* stream) {
    if (!dtype_ok(dtype) || rows < 0 || m < 1 || m > 256 || ldi < m || ldo < m ||
        (rows > 0 && (src == nullptr || perm == nullptr || out == nullptr || bad == nullptr)))
        return fail(SDB_EINVAL, "sdb_ingest_gather: bad args");
    int rc = dtype == SDB_F64 ? sdb::ingest_gather<double>(rows, (int)m, src, ldi, perm, (double*)out, ldo, bad, S(stream))
                              : sdb::ingest_gather<float>(rows, (int)m, src, ldi, perm, (float*)out, ldo, bad, S(stream));
    return cuda_rc(rc, "sdb_ingest_gather");
}

int sdb_ingest_gather_split(int dtype, int64_t rows, int64_t m, const double* src, int64_t ldi,
                            const int64_t* perm, const double* dsrc, int64_t drows, void* out, int64_t ldo,
                            int32_t* bad, void* stream) {
    if (!dtype_ok(dtype) || rows < 0 || m < 1 || m > 256 || ldi < m || ldo < m || drows < 0 ||
        (drows > 0 && dsrc == nullptr) ||
        (rows > 0 && (src == nullptr || perm == nullptr || out == nullptr || bad == nullptr)))
        return fail(SDB_EINVAL, "sdb_ingest_gather_split: bad args");
    int rc = dtype == SDB_F64
                 ? sdb::ingest_gather<double>(rows, (int)m, src, ldi, perm, (double*)out, ldo, bad, S(stream), dsrc, drows)
                 : sdb::ingest_gather<float>(rows, (int)m, src, ldi, perm, (float*)out, ldo, bad, S(stream), dsrc, drows);
    return cuda_rc(rc, "sdb_ingest_gather_split");
}

int sdb_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
    if (bytes < 0 || (bytes > 0 && (dst == nullptr || src == nullptr)))
        return fail(SDB_EINVAL, "sdb_copy_async: bad args");
    if (bytes == 0) return SDB_OK;
    return cuda_rc((int)cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, S(stream)), "sdb_copy_async");
}

int sdb_host_mapped(const void* host, void** dev) {
    if (host == nullptr || dev == nullptr) return fail(SDB_EINVAL, "sdb_host_mapped: bad args");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return fail(SDB_EINVAL, "sdb_host_mapped: not a CUDA host allocation");
    }
    if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr)
        return fail(SDB_EINVAL, "sdb_host_mapped: not pinned, device-mapped host memory");
    *dev = at.devicePointer;
    return SDB_OK;
}

int sdb_csc_to_codes(int dtype, int64_t N, int64_t cap, const int64_t* indptr,
                     const int64_t* indices, const double* data, int32_t* idx, void* val,
                     int32_t* counts, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || cap < 1) return fail(SDB_EINVAL, "sdb_csc_to_codes: bad args");
    int rc = dtype == SDB_F64 ? sdb::csc_to_codes<double>(N, (int)cap, indptr, indices, data, idx, (double*)val, counts, S(stream))
                              : sdb::csc_to_codes<float>(N, (int)cap, indptr, indices, data, idx, (float*)val, counts, S(stream));
    return cuda_rc(rc, "sdb_csc_to_codes");
}

int sdb_normalize(int64_t rows, int64_t m, const double* in, double* out, double* scales, void* stream) {
    if (rows < 0 || m < 1) return fail(SDB_EINVAL, "sdb_normalize: bad args");
    return cuda_rc(sdb::normalize_rows(rows, (int)m, in, out, scales, S(stream)), "sdb_normalize");
}

int sdb_synth_sparse(int dtype, int64_t N, int64_t m, int64_t K, int64_t s, const double* D, double sigma,
                     uint64_t seed, void* Y, int64_t ldy, int32_t* sup_out, void* stream) {
    if (!dtype_ok(dtype) || N < 0 || m < 1 || K < 1 || s < 1 || s > K || s > 64 || ldy < m || !(sigma >= 0.0))
        return fail(SDB_EINVAL, "sdb_synth_sparse: bad args");
    return cuda_rc(sdb::synth_sparse(dtype == SDB_F64, N, (int)m, (int)K, (int)s, D, sigma, seed, Y, ldy, sup_out,
                                     S(stream)),
                   "sdb_synth_sparse");
}

int sdb_extract_patches(int dtype, const double* img, int64_t H, int64_t W, int64_t p, int64_t s,
                        void* out, void* stream) {
    if (!dtype_ok(dtype) || p < 1 || s < 1 || p > H || p > W) return fail(SDB_EINVAL, "sdb_extract_patches: bad args");
    int rc = dtype == SDB_F64 ? sdb::extract_patches<double>(img, (int)H, (int)W, (int)p, (int)s, (double*)out, S(stream))
                              : sdb::extract_patches<float>(img, (int)H, (int)W, (int)p, (int)s, (float*)out, S(stream));
    return cuda_rc(rc, "sdb_extract_patches");
}

int sdb_reconstruct(int dtype, int64_t H, int64_t W, int64_t p, int64_t s, const double* D,
                    int64_t cap, const int32_t* idx, const void* val, const int32_t* counts,
                    double lo, double hi, double* out, void* stream) {
    if (!dtype_ok(dtype) || p < 1 || s < 1 || p > H || p > W || cap < 1) return fail(SDB_EINVAL, "sdb_reconstruct: bad args");
    int rc = dtype == SDB_F64
                 ? sdb::reconstruct<double>((int)H, (int)W, (int)p, (int)s, D, (int)cap, idx, (const double*)val, counts, lo, hi, out, S(stream))
                 : sdb::reconstruct<float>((int)H, (int)W, (int)p, (int)s, D, (int)cap, idx, (const float*)val, counts, lo, hi, out, S(stream));
    return cuda_rc(rc, "sdb_reconstruct");
}

int sdb_reconstruct_dense(int64_t H, int64_t W, int64_t p, int64_t s, const double* P, double* out,
                          void* stream) {
    if (p < 1 || s < 1 || p > H || p > W) return fail(SDB_EINVAL, "sdb_reconstruct_dense: bad args");
    return cuda_rc(sdb::reconstruct_dense((int)H, (int)W, (int)p, (int)s, P, out, S(stream)), "sdb_reconstruct_dense");
}

}  // extern "C"
