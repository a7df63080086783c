// Data-movement and patch-pipeline kernels around the OMP/MOD core.
//
// Reference: denoising.py:118-163,223-239 (patch extraction, overlap
// averaging, clip), trainer.py:200-223 (shard gather), sparse_coding.py:76-133
// (CSC container -> per-signal code rows), dictionary_update.py:56-69
// (normalize_columns).
#include <algorithm>

#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_aux.h"

namespace sdb {

// out[r] = in[perm[r]] for rows of length m (split_dataset's column gather)
template <typename T>
__global__ void k_gather_rows(int64_t rows, int m, const T* __restrict__ in, int64_t ldi,
                              const int64_t* __restrict__ perm, T* __restrict__ out, int64_t ldo) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= rows) return;
    const T* src = in + perm[r] * ldi;
    T* dst = out + r * ldo;
    for (int t = lane; t < m; t += 32) dst[t] = src[t];
}

// out[r] = (T) src[perm[r]] for f64 rows of length m, with a non-finite flag:
// the split's gather fused with the input cast and the finiteness check. src
// may be device memory or pinned, device-mapped host memory (the rows then
// cross PCIe in permuted order); each warp keeps U rows in flight.
template <typename T, int MPL, int U>
__global__ void __launch_bounds__(256)
k_ingest_gather(int64_t rows, int m, const double* __restrict__ src, int64_t ldi, const int64_t* __restrict__ perm,
                T* __restrict__ out, int64_t ldo, int32_t* __restrict__ bad, const double* __restrict__ dsrc,
                int64_t drows) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * wpb;
    bool nonfinite = false;
    for (int64_t r0 = ((int64_t)blockIdx.x * wpb + (threadIdx.x >> 5)) * U; r0 < rows; r0 += nw * U) {
        double v[U][MPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + u;
            const int64_t pr = r < rows ? perm[r] : 0;
            // source rows below drows were copied to the device beforehand
            const double* row = pr < drows ? dsrc + pr * ldi : src + pr * ldi;
#pragma unroll
            for (int q = 0; q < MPL; ++q) {
                const int t = lane + 32 * q;
                v[u][q] = (r < rows && t < m) ? row[t] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + u;
            if (r >= rows) break;
#pragma unroll
            for (int q = 0; q < MPL; ++q) {
                const int t = lane + 32 * q;
                if (t < m) {
                    nonfinite |= !isfinite(v[u][q]);
                    out[r * ldo + t] = (T)v[u][q];
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) *bad = 1;
}

template <typename T, int MPL>
static void launch_gather(bool host, int64_t rows, int m, const double* src, int64_t ldi, const int64_t* perm,
                          T* out, int64_t ldo, int32_t* bad, const double* dsrc, int64_t drows, cudaStream_t st) {
    if (host) {
        // pinned host source: 64 CTAs keep ~2K rows (~1 MB) in flight, plenty
        // for PCIe, and leave the SMs to concurrently running training kernels
        // (measured: one 2-warp CTA per SM reads PCIe ~15% slower)
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 31) / 32, 64));
        k_ingest_gather<T, MPL, 4><<<g, 256, 0, st>>>(rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows);
    } else {
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 31) / 32, 148 * 16));
        k_ingest_gather<T, MPL, 4><<<g, 256, 0, st>>>(rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows);
    }
}

template <typename T>
int ingest_gather(int64_t rows, int m, const double* src, int64_t ldi, const int64_t* perm, T* out, int64_t ldo,
                  int32_t* bad, cudaStream_t st, const double* dsrc, int64_t drows) {
    if (rows <= 0) return 0;
    cudaPointerAttributes at{};
    const bool host = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const int mpl = (m + 31) / 32;
    if (mpl <= 1) launch_gather<T, 1>(host, rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows, st);
    else if (mpl <= 2) launch_gather<T, 2>(host, rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows, st);
    else if (mpl <= 5) launch_gather<T, 5>(host, rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows, st);
    else launch_gather<T, 8>(host, rows, m, src, ldi, perm, out, ldo, bad, dsrc, drows, st);
    return (int)cudaGetLastError();
}
template int ingest_gather<float>(int64_t, int, const double*, int64_t, const int64_t*, float*, int64_t, int32_t*,
                                  cudaStream_t, const double*, int64_t);
template int ingest_gather<double>(int64_t, int, const double*, int64_t, const int64_t*, double*, int64_t,
                                   int32_t*, cudaStream_t, const double*, int64_t);

// CSC (indptr, indices, data) -> codes rows (idx N x cap, val, counts)
template <typename T>
__global__ void k_csc_to_codes(int64_t N, int cap, const int64_t* __restrict__ indptr,
                               const int64_t* __restrict__ indices, const double* __restrict__ data,
                               int32_t* __restrict__ idx, T* __restrict__ val, int32_t* __restrict__ counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t a = indptr[i], b = indptr[i + 1];
    const int n = (int)(b - a);
    counts[i] = n;
    for (int t = 0; t < cap; ++t) {
        idx[i * cap + t] = t < n ? (int32_t)indices[a + t] : 0;
        val[i * cap + t] = t < n ? (T)data[a + t] : T(0);
    }
}

// rows of length m: out = row / ||row|| (zero rows untouched), scales = norms
__global__ void k_normalize(int64_t rows, int m, const double* __restrict__ in, double* __restrict__ out,
                            double* __restrict__ scales) {
    const int lane = threadIdx.x & 31;
    const int64_t a = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (a >= rows) return;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(in[a * m + r], in[a * m + r], s);
    const double nrm = sqrt(warp_sum(s));
    for (int r = lane; r < m; r += 32) out[a * m + r] = nrm > 0.0 ? in[a * m + r] / nrm : in[a * m + r];
    if (lane == 0 && scales) scales[a] = nrm;
}

// all p x p windows at stride s, column-major vectorised, row-offset major
// order (denoising.py:118-135): patch k = r*C + c, element i + j*p
template <typename T>
__global__ void k_extract(const double* __restrict__ img, int H, int W, int p, int s, int R, int C,
                          T* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t pp = (int64_t)p * p;
    if (e >= (int64_t)R * C * pp) return;
    const int64_t k = e / pp;
    const int q = (int)(e % pp);
    const int i = q % p, j = q / p;
    const int r = (int)(k / C), c = (int)(k % C);
    out[e] = (T)img[(int64_t)(r * s + i) * W + (c * s + j)];
}

// overlap averaging of the patch estimates D x_k (denoising.py:138-163,236-239)
// as a gather: each pixel sums its covering patches in the reference's
// (column offset j, row offset i) order, divides by the count, clips.
template <typename T>
__global__ void k_reconstruct(int H, int W, int p, int s, int R, int C, const double* __restrict__ D,
                              int m, int cap, const int32_t* __restrict__ idx, const T* __restrict__ val,
                              const int32_t* __restrict__ counts, double lo, double hi,
                              double* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)H * W) return;
    const int y = (int)(e / W), x = (int)(e % W);
    double sum = 0.0, cnt = 0.0;
    for (int j = 0; j < p; ++j) {
        const int cx = x - j;
        if (cx < 0 || cx % s) continue;
        const int c = cx / s;
        if (c >= C) continue;
        for (int i = 0; i < p; ++i) {
            const int ry = y - i;
            if (ry < 0 || ry % s) continue;
            const int r = ry / s;
            if (r >= R) continue;
            const int64_t k = (int64_t)r * C + c;
            const int n = counts[k];
            const int row = i + j * p;
            double est = 0.0;
            for (int t = 0; t < n; ++t)
                est = fma(D[(int64_t)idx[k * cap + t] * m + row], (double)val[k * cap + t], est);
            sum += est;
            cnt += 1.0;
        }
    }
    double v = cnt > 0.0 ? sum / cnt : 0.0;
    out[e] = fmin(fmax(v, lo), hi);
}

// reconstruct_from_patches on an explicit estimate matrix (n x p^2, signal-major)
__global__ void k_reconstruct_dense(int H, int W, int p, int s, int R, int C, const double* __restrict__ P,
                                    double* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)H * W) return;
    const int y = (int)(e / W), x = (int)(e % W);
    double sum = 0.0, cnt = 0.0;
    for (int j = 0; j < p; ++j) {
        const int cx = x - j;
        if (cx < 0 || cx % s) continue;
        const int c = cx / s;
        if (c >= C) continue;
        for (int i = 0; i < p; ++i) {
            const int ry = y - i;
            if (ry < 0 || ry % s) continue;
            const int r = ry / s;
            if (r >= R) continue;
            sum += P[((int64_t)r * C + c) * p * p + i + j * p];
            cnt += 1.0;
        }
    }
    out[e] = cnt > 0.0 ? sum / cnt : 0.0;
}

int reconstruct_dense(int H, int W, int p, int s, const double* P, double* out, cudaStream_t st) {
    const int R = (H - p) / s + 1, C = (W - p) / s + 1;
    const int64_t n = (int64_t)H * W;
    k_reconstruct_dense<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, W, p, s, R, C, P, out);
    return (int)cudaGetLastError();
}

// 16-byte row pieces: a half-warp per row (lane l of the half moves 16-byte
// piece l, l + 16, ...), each warp keeps 8 rows (4 row pairs) in flight
template <int PPL>
__global__ void __launch_bounds__(256)
k_gather_rows_v4(int64_t rows, int pieces, const float4* __restrict__ in, int64_t ldi4,
                 const int64_t* __restrict__ perm, float4* __restrict__ out, int64_t ldo4) {
    const int lane = threadIdx.x & 31, h = lane >> 4, l16 = lane & 15;
    const int64_t r0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 8;
    int64_t src[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t r = r0 + 2 * u + h;
        src[u] = r < rows ? perm[r] : -1;
    }
    float4 v[4][PPL];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < PPL; ++q) {
            const int pc = l16 + 16 * q;
            if (src[u] >= 0 && pc < pieces) v[u][q] = __ldg(in + src[u] * ldi4 + pc);
        }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t r = r0 + 2 * u + h;
#pragma unroll
        for (int q = 0; q < PPL; ++q) {
            const int pc = l16 + 16 * q;
            if (src[u] >= 0 && pc < pieces) out[r * ldo4 + pc] = v[u][q];
        }
    }
}

template <typename T>
int gather_rows(int64_t rows, int m, const T* in, int64_t ldi, const int64_t* perm, T* out, int64_t ldo,
                cudaStream_t st) {
    if (rows <= 0) return 0;
    const int64_t bytes = (int64_t)m * sizeof(T);
    const bool v4 = bytes % 16 == 0 && (ldi * (int64_t)sizeof(T)) % 16 == 0 && (ldo * (int64_t)sizeof(T)) % 16 == 0 &&
                    ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0 && bytes <= 2048;
    if (v4) {
        const int pieces = (int)(bytes / 16);
        const int64_t ldi4 = ldi * (int64_t)sizeof(T) / 16, ldo4 = ldo * (int64_t)sizeof(T) / 16;
        const unsigned g = (unsigned)((rows + 63) / 64);
        const float4* i4 = reinterpret_cast<const float4*>(in);
        float4* o4 = reinterpret_cast<float4*>(out);
        if (pieces <= 16) k_gather_rows_v4<1><<<g, 256, 0, st>>>(rows, pieces, i4, ldi4, perm, o4, ldo4);
        else if (pieces <= 32) k_gather_rows_v4<2><<<g, 256, 0, st>>>(rows, pieces, i4, ldi4, perm, o4, ldo4);
        else if (pieces <= 64) k_gather_rows_v4<4><<<g, 256, 0, st>>>(rows, pieces, i4, ldi4, perm, o4, ldo4);
        else k_gather_rows_v4<8><<<g, 256, 0, st>>>(rows, pieces, i4, ldi4, perm, o4, ldo4);
        return (int)cudaGetLastError();
    }
    k_gather_rows<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, m, in, ldi, perm, out, ldo);
    return (int)cudaGetLastError();
}
template int gather_rows<float>(int64_t, int, const float*, int64_t, const int64_t*, float*, int64_t, cudaStream_t);
template int gather_rows<double>(int64_t, int, const double*, int64_t, const int64_t*, double*, int64_t, cudaStream_t);

template <typename T>
int csc_to_codes(int64_t N, int cap, const int64_t* indptr, const int64_t* indices, const double* data,
                 int32_t* idx, T* val, int32_t* counts, cudaStream_t st) {
    if (N <= 0) return 0;
    k_csc_to_codes<T><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, cap, indptr, indices, data, idx, val, counts);
    return (int)cudaGetLastError();
}
template int csc_to_codes<float>(int64_t, int, const int64_t*, const int64_t*, const double*, int32_t*, float*, int32_t*, cudaStream_t);
template int csc_to_codes<double>(int64_t, int, const int64_t*, const int64_t*, const double*, int32_t*, double*, int32_t*, cudaStream_t);

int normalize_rows(int64_t rows, int m, const double* in, double* out, double* scales, cudaStream_t st) {
    if (rows <= 0) return 0;
    k_normalize<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, m, in, out, scales);
    return (int)cudaGetLastError();
}

template <typename T>
int extract_patches(const double* img, int H, int W, int p, int s, T* out, cudaStream_t st) {
    const int R = (H - p) / s + 1, C = (W - p) / s + 1;
    const int64_t n = (int64_t)R * C * p * p;
    if (n <= 0) return 0;
    k_extract<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(img, H, W, p, s, R, C, out);
    return (int)cudaGetLastError();
}
template int extract_patches<float>(const double*, int, int, int, int, float*, cudaStream_t);
template int extract_patches<double>(const double*, int, int, int, int, double*, cudaStream_t);

template <typename T>
int reconstruct(int H, int W, int p, int s, const double* D, int cap, const int32_t* idx, const T* val,
                const int32_t* counts, double lo, double hi, double* out, cudaStream_t st) {
    const int R = (H - p) / s + 1, C = (W - p) / s + 1;
    const int64_t n = (int64_t)H * W;
    k_reconstruct<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, W, p, s, R, C, D, p * p, cap, idx,
                                                                 val, counts, lo, hi, out);
    return (int)cudaGetLastError();
}
template int reconstruct<float>(int, int, int, int, const double*, int, const int32_t*, const float*, const int32_t*, double, double, double*, cudaStream_t);
template int reconstruct<double>(int, int, int, int, const double*, int, const int32_t*, const double*, const int32_t*, double, double, double*, cudaStream_t);

}  // namespace sdb
