// C-ABI entry points (include/sparsedict_b200.h). Validation of sizes and
// dtypes happens here; data-dependent preconditions (unit-norm dictionary,
// finite inputs, mode choice) are checked by the Python boundary before any
// launch, as the reference does (sparse_coding.py:145-155, 241-264).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/sparsedict_b200.h"
#include "sdb_common.cuh"
#include "sdb_internal.h"

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

int sdb_abi_version(void) { return 1; }
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

int sdb_correlate(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off,
                  int64_t max_shard_rows, const void* Y, int64_t ldy, const void* D, void* alpha0,
                  int64_t lda, int use_tc, void* stream) {
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
            rc = sdb::correlate_tc_f32((const float*)Y, ldy, shard_off, max_shard_rows, (int)P,
                                       (const float*)D, m, K, (float*)alpha0, lda, S(stream));
        if (rc == cudaErrorNotSupported)
            rc = sdb::correlate_simt_f32((const float*)Y, ldy, shard_off, max_shard_rows, (int)P,
                                         (const float*)D, m, K, (float*)alpha0, lda, S(stream));
    }
    return cuda_rc(rc, "sdb_correlate");
}

int64_t sdb_omp_scratch_bytes(int dtype, int64_t N, int64_t m, int64_t cap) {
    if (!dtype_ok(dtype) || cap < 1 || m < 1) return fail(SDB_EINVAL, "sdb_omp_scratch_bytes: bad args");
    const int64_t wb = dtype == SDB_F64 ? sdb::omp_warp_bytes_f64((int)cap, (int)m)
                                        : sdb::omp_warp_bytes_f32((int)cap, (int)m);
    if (wb * 8 <= 200 * 1024) return 0;  // fits shared memory
    const int64_t warps = std::max<int64_t>(8, std::min<int64_t>(((N + 7) / 8) * 8, (int64_t)148 * 32));
    return wb * warps;
}

int sdb_omp(int dtype, int64_t N, int64_t m, int64_t K, int64_t P, const int64_t* shard_off,
            const void* alpha0, int64_t lda, const void* Y, int64_t ldy, const void* D,
            const void* G, int64_t cap, double eps, double guard, int32_t* idx, void* val,
            int32_t* counts, int8_t* status, void* rnorm, void* scratch, int64_t scratch_bytes,
            void* stream) {
    if (!dtype_ok(dtype) || N < 0 || m < 1 || K < 1 || P < 1 || cap < 1 || ldy < m || lda < K)
        return fail(SDB_EINVAL, "sdb_omp: bad args");
    if (K > 1024) return fail(SDB_EINVAL, "sdb_omp: K=%lld > 1024 not supported", (long long)K);
    if (N == 0) return SDB_OK;
    const int64_t wb = dtype == SDB_F64 ? sdb::omp_warp_bytes_f64((int)cap, (int)m)
                                        : sdb::omp_warp_bytes_f32((int)cap, (int)m);
    const bool need_global = wb * 8 > 200 * 1024;
    if (need_global && (scratch == nullptr || scratch_bytes < wb * 8))
        return fail(SDB_EINVAL, "sdb_omp: scratch of %lld bytes required", (long long)(wb * 8));
    auto fill = [&](auto& a) {
        a.N = N; a.m = (int)m; a.K = (int)K; a.cap = (int)cap; a.P = (int)P;
        a.shard_off = shard_off; a.lda = lda; a.ldy = ldy;
        a.idx = idx; a.counts = counts; a.status = status;
        a.gscratch = need_global ? (unsigned char*)scratch : nullptr;
        a.gscratch_warps = need_global ? scratch_bytes / wb : 0;
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
        rc = sdb::launch_omp<float>(a, S(stream));
    }
    return cuda_rc(rc, "sdb_omp");
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

}  // extern "C"
