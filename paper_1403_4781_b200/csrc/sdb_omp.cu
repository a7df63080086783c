// Batch-OMP on B200: correlation / Gram products, the warp-per-signal greedy
// kernel and CSC packing.
//
// Reference: /root/reference/pkg/src/sparsedict/_kernels.py:23-173 (Numba
// kernels) and sparse_coding.py:266-303 (Gram per call, batch loop, packing).
//
// Device layouts:
//   Y      : N x ldy, signal-major (row i = signal i, m contiguous)  [= F-order m x N]
//   D      : P x K x m, atom-major per shard                          [= F-order m x K]
//   G      : P x K x K
//   alpha0 : N x lda   (alpha0[i, j] = <d_j, y_i>, shard of i)
//   codes  : idx N x cap (int32, selection order), val N x cap, counts, status, rnorm
#include "sdb_common.cuh"
#include "sdb_internal.h"

namespace sdb {

// ----------------------------------------------------------------------------
// Row-dot tile kernel:  C[a, b] = sum_t A[a, t] * B_p[b, t]  (t ascending).
// Used for the exact FP64 correlation alpha0 = Y D (per shard) and for every
// Gram matrix G = D^T D (A = B = D_p). In exact mode each output is a
// sequential sum over t with separately rounded products, matching
// _kernels.py:23-35 / :54-59 bit for bit.
// ----------------------------------------------------------------------------
constexpr int RD_BM = 64, RD_BN = 64, RD_BK = 16;

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256)
k_rowdot(const TIn* __restrict__ A, int64_t lda, const int64_t* __restrict__ a_off,
         int64_t a_rows_per_shard, const TIn* __restrict__ B, int64_t ldb, int64_t b_stride,
         int64_t nb, int64_t kdim, TOut* __restrict__ C, int64_t ldc, bool sym,
         float* __restrict__ C32 = nullptr) {
    // sym (Gram, A == B per shard): only tiles on or above the diagonal are
    // computed; an upper tile also writes its mirror (products commute, so the
    // mirrored entry is bitwise the one its own tile would compute)
    if (sym && blockIdx.y < blockIdx.x) return;
    using R = Ar<TIn>;
    __shared__ TIn As[RD_BK][RD_BM + 1];
    __shared__ TIn Bs[RD_BK][RD_BN + 1];
    const int p = blockIdx.z;
    const int64_t a_lo = a_off ? a_off[p] : (int64_t)p * a_rows_per_shard;
    const int64_t a_hi = a_off ? a_off[p + 1] : a_lo + a_rows_per_shard;
    const int64_t a0 = a_lo + (int64_t)blockIdx.x * RD_BM;
    if (a0 >= a_hi) return;
    const int64_t b0 = (int64_t)blockIdx.y * RD_BN;
    if (b0 >= nb) return;
    const TIn* Bp = B + (int64_t)p * b_stride;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    TIn acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = TIn(0);

    for (int64_t k0 = 0; k0 < kdim; k0 += RD_BK) {
        // cooperative loads: 64 rows x 16 k for each operand (4 per thread)
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int e = threadIdx.x + l * 256;
            const int row = e >> 4, kk = e & 15;
            const int64_t ga = a0 + row, gb = b0 + row, gk = k0 + kk;
            As[kk][row] = (ga < a_hi && gk < kdim) ? A[ga * lda + gk] : TIn(0);
            Bs[kk][row] = (gb < nb && gk < kdim) ? Bp[gb * ldb + gk] : TIn(0);
        }
        __syncthreads();
        const int kend = (int)((kdim - k0) < RD_BK ? (kdim - k0) : RD_BK);
        for (int kk = 0; kk < kend; ++kk) {
            TIn av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = R::mac(acc[i][j], av[i], bv[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t ga = a0 + ty + 16 * i;
        if (ga >= a_hi) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gb = b0 + tx + 16 * j;
            if (gb < nb) {
                C[ga * ldc + gb] = (TOut)acc[i][j];
                if (sym && blockIdx.y > blockIdx.x) C[(a_lo + gb) * ldc + (ga - a_lo)] = (TOut)acc[i][j];
                if (C32 != nullptr) {   // the same sums rounded once to FP32 (the coding kernels' copy)
                    C32[ga * ldc + gb] = (float)acc[i][j];
                    if (sym && blockIdx.y > blockIdx.x) C32[(a_lo + gb) * ldc + (ga - a_lo)] = (float)acc[i][j];
                }
            }
        }
    }
}

template <typename TIn, typename TOut>
static int launch_rowdot(const TIn* A, int64_t lda, const int64_t* a_off, int64_t a_rows_max,
                         int64_t a_rows_per_shard, const TIn* B, int64_t ldb, int64_t b_stride,
                         int64_t nb, int64_t kdim, TOut* C, int64_t ldc, int P,
                         cudaStream_t st, bool sym = false, float* C32 = nullptr) {
    if (a_rows_max <= 0 || nb <= 0 || P <= 0) return 0;
    dim3 grid((unsigned)((a_rows_max + RD_BM - 1) / RD_BM), (unsigned)((nb + RD_BN - 1) / RD_BN),
              (unsigned)P);
    k_rowdot<TIn, TOut><<<grid, 256, 0, st>>>(A, lda, a_off, a_rows_per_shard, B, ldb, b_stride,
                                              nb, kdim, C, ldc, sym, C32);
    return (int)cudaGetLastError();
}

// G64 = D^T D in FP64 and G32 = (float)G64 from one pass (gram_f32 rounds the
// same FP64 sums, so G32 is bitwise gram_f32's)
int gram_f64_f32(const double* D, int P, int64_t m, int64_t K, double* G64, float* G32, cudaStream_t st) {
    return launch_rowdot<double, double>(D, m, nullptr, K, K, D, m, K * m, K, m, G64, K, P, st, true, G32);
}
// FP32 Gram of FP32 rows (a screening pass: atom-pair coherences to ~1e-5)
int gram_screen_f32(const float* D, int P, int64_t m, int64_t K, float* G, cudaStream_t st) {
    return launch_rowdot<float, float>(D, m, nullptr, K, K, D, m, K * m, K, m, G, K, P, st, true);
}
int gram_f64(const double* D, int P, int64_t m, int64_t K, double* G, cudaStream_t st) {
    return launch_rowdot<double, double>(D, m, nullptr, K, K, D, m, K * m, K, m, G, K, P, st, true);
}
int gram_f32(const double* D, int P, int64_t m, int64_t K, float* G, cudaStream_t st) {
    return launch_rowdot<double, float>(D, m, nullptr, K, K, D, m, K * m, K, m, G, K, P, st, true);
}
int correlate_simt_f64(const double* Y, int64_t ldy, const int64_t* off, int64_t max_rows, int P,
                       const double* D, int64_t m, int64_t K, double* alpha, int64_t lda,
                       cudaStream_t st) {
    return launch_rowdot<double, double>(Y, ldy, off, max_rows, 0, D, m, K * m, K, m, alpha, lda,
                                         P, st);
}
int correlate_simt_f32(const float* Y, int64_t ldy, const int64_t* off, int64_t max_rows, int P,
                       const float* D, int64_t m, int64_t K, float* alpha, int64_t lda,
                       cudaStream_t st) {
    return launch_rowdot<float, float>(Y, ldy, off, max_rows, 0, D, m, K * m, K, m, alpha, lda, P,
                                       st);
}

// ----------------------------------------------------------------------------
// Greedy OMP, one warp per signal.
//
// Lane l owns atoms j = l + 32k (k < KPL): c0 and corr live in registers.
// Per step (reference _kernels.py:78-154):
//   corr = c0 - sum_t G[idx_t, :] x_t  (G rows streamed through L2, coalesced)
//   |.|, support exclusion, warp max, stall test, lowest index in tie window
//   Cholesky append with the diagonal guard, forward/back substitution,
//   explicit residual r = y - D_S x and its norm.
// Exact mode (double) runs the O(n^2) recurrences in the reference's order on
// every lane (identical values, no divergence); fast mode (float) uses
// lane-parallel column sweeps when the support fits one warp (cap <= 32).
// ----------------------------------------------------------------------------
template <typename T>
struct WarpScratch {
    T* L;      // packed lower-triangular Cholesky factor, row t at t(t+1)/2
    T* tmp;    // forward-substitution vector
    T* x;      // coefficients (support order)
    T* y;      // signal
    T* r;      // residual
    int* ids;  // support (selection order)
};

__host__ __device__ inline int64_t align16(int64_t b) { return (b + 15) & ~int64_t(15); }

template <typename T>
__host__ __device__ inline int64_t omp_warp_bytes(int cap, int m) {
    int64_t b = align16(sizeof(T) * ((int64_t)cap * (cap + 1) / 2));
    b += align16(sizeof(T) * cap) * 2;
    b += align16(sizeof(T) * m) * 2;
    b += align16(sizeof(int) * cap);
    return b;
}

template <typename T>
__device__ inline WarpScratch<T> carve(unsigned char* base, int cap, int m) {
    WarpScratch<T> w;
    unsigned char* p = base;
    w.L = (T*)p;   p += align16(sizeof(T) * ((int64_t)cap * (cap + 1) / 2));
    w.tmp = (T*)p; p += align16(sizeof(T) * cap);
    w.x = (T*)p;   p += align16(sizeof(T) * cap);
    w.y = (T*)p;   p += align16(sizeof(T) * m);
    w.r = (T*)p;   p += align16(sizeof(T) * m);
    w.ids = (int*)p;
    return w;
}

template <typename T>
__device__ __forceinline__ const T* tri_row(const T* L, int t) { return L + (int64_t)t * (t + 1) / 2; }
template <typename T>
__device__ __forceinline__ T* tri_row(T* L, int t) { return L + (int64_t)t * (t + 1) / 2; }

template <typename T, int KPL>
__global__ void __launch_bounds__(256)
k_omp(OmpArgs<T> a) {
    using R = Ar<T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * wpb + wib;
    const int64_t nw = (int64_t)gridDim.x * wpb;
    unsigned char* base = a.gscratch ? a.gscratch + gw * a.warp_bytes : smem + wib * a.warp_bytes;
    WarpScratch<T> w = carve<T>(base, a.cap, a.m);
    const int m = a.m, K = a.K, cap = a.cap;
    const T eps = a.eps;

    const int64_t n_items = a.list ? ((int64_t)*a.nlist < a.N ? (int64_t)*a.nlist : a.N) : a.N;
    for (int64_t e = gw; e < n_items; e += nw) {
        const int64_t i = a.list ? (int64_t)a.list[e] : e;
        const int p = shard_of(a.shard_off, a.P, i);
        const T* __restrict__ Gp = a.G + (int64_t)p * K * K;
        const T* __restrict__ Dp = a.D + (int64_t)p * K * m;
        if (a.Yf) {
            for (int t = lane; t < m; t += 32) w.y[t] = (T)a.Yf[i * a.ldy + t];
        } else {
            for (int t = lane; t < m; t += 32) w.y[t] = a.Y[i * a.ldy + t];
        }
        __syncwarp();
        T c0[KPL];
        if (a.alpha0) {
#pragma unroll
            for (int k = 0; k < KPL; ++k) {
                const int j = lane + 32 * k;
                c0[k] = (j < K) ? a.alpha0[i * a.lda + j] : T(0);
            }
        } else {
            // c0 = D^T y with the reference's loop order (sequential over the
            // m rows, separately rounded products: _kernels.py:54-59)
            if (a.Dt) {
                // transposed copy: lanes read consecutive atoms of one row t
                const T* __restrict__ Dtp = a.Dt + (int64_t)p * m * K;
#pragma unroll
                for (int k = 0; k < KPL; ++k) c0[k] = T(0);
                for (int t = 0; t < m; ++t) {
                    const T yt = w.y[t];
#pragma unroll
                    for (int k = 0; k < KPL; ++k) {
                        const int j = lane + 32 * k;
                        if (j < K) c0[k] = R::mac(c0[k], __ldg(Dtp + (int64_t)t * K + j), yt);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < KPL; ++k) {
                    const int j = lane + 32 * k;
                    T acc = T(0);
                    if (j < K) {
                        const T* __restrict__ dj = Dp + (int64_t)j * m;
                        for (int t = 0; t < m; ++t) acc = R::mac(acc, __ldg(dj + t), w.y[t]);
                    }
                    c0[k] = acc;
                }
            }
        }
        T ysq;
        if constexpr (R::kExact) {
            ysq = T(0);
            for (int t = 0; t < m; ++t) ysq = R::mac(ysq, w.y[t], w.y[t]);
        } else {
            T part = T(0);
            for (int t = lane; t < m; t += 32) part = fmaf(w.y[t], w.y[t], part);
            ysq = warp_sum(part);
        }
        T rnorm = R::sqrt_(ysq);
        int n = 0;
        int status = 0;
        if (!(rnorm <= eps || rnorm == T(0))) {
            uint32_t selbits = 0;  // bit k: atom lane+32k is in the support
            for (int step = 0; step < cap; ++step) {
                // ---- correlations of the current residual (_kernels.py:81-96)
                T corr[KPL];
#pragma unroll
                for (int k = 0; k < KPL; ++k) corr[k] = c0[k];
                for (int t = 0; t < n; ++t) {
                    const T coef = w.x[t];
                    const T* __restrict__ g = Gp + (int64_t)w.ids[t] * K;
#pragma unroll
                    for (int k = 0; k < KPL; ++k) {
                        const int j = lane + 32 * k;
                        if (j < K) corr[k] = R::msub(corr[k], __ldg(g + j), coef);
                    }
                }
                T lmax = T(-1);
#pragma unroll
                for (int k = 0; k < KPL; ++k) {
                    const int j = lane + 32 * k;
                    const bool ok = (j < K) && !((selbits >> k) & 1u);
                    const T av = ok ? fabs(corr[k]) : T(-1);
                    corr[k] = av;
                    lmax = fmax(lmax, av);
                }
                const T cmax = warp_max(lmax);
                if (cmax <= R::mul(T(1e-13), rnorm)) {  // _kernels.py:97-100
                    status = 3;
                    break;
                }
                const T thresh = R::sub(cmax, R::mul(T(1e-12), cmax));
                int cand = 0x7fffffff;
#pragma unroll
                for (int k = KPL - 1; k >= 0; --k)
                    if (corr[k] >= thresh) cand = lane + 32 * k;  // lowest k wins
                const int best = warp_min_int(cand);

                // ---- Cholesky append (_kernels.py:109-127)
                T* Lrow = tri_row(w.L, n);
                T dsq = __ldg(Gp + (int64_t)best * K + best);
                if (R::kExact || n > 32) {
                    for (int t = 0; t < n; ++t) {
                        T acc = __ldg(Gp + (int64_t)w.ids[t] * K + best);
                        const T* Lt = tri_row(w.L, t);
                        for (int u = 0; u < t; ++u) acc = R::msub(acc, Lt[u], Lrow[u]);
                        const T wv = R::div(acc, Lt[t]);
                        Lrow[t] = wv;  // every lane writes the same value
                        dsq = R::msub(dsq, wv, wv);
                    }
                } else {
                    // lane-parallel column sweep: lane t solves for w_t
                    T acc = (lane < n) ? __ldg(Gp + (int64_t)w.ids[lane] * K + best) : T(0);
                    T mine = T(0);
                    for (int u = 0; u < n; ++u) {
                        const T wu = R::div(__shfl_sync(SDB_FULL, acc, u), tri_row(w.L, u)[u]);
                        if (lane == u) mine = wu;
                        if (lane > u && lane < n) acc = R::msub(acc, tri_row(w.L, lane)[u], wu);
                    }
                    if (lane < n) Lrow[lane] = mine;
                    dsq = R::sub(dsq, warp_sum(lane < n ? mine * mine : T(0)));
                }
                if (dsq <= a.guard) {  // numerically singular support Gram
                    status = 2;
                    break;
                }
                __syncwarp();
                if (lane == 0) {
                    Lrow[n] = R::sqrt_(dsq);
                    w.ids[n] = best;
                }
                if (lane == (best & 31)) selbits |= 1u << (best >> 5);
                // c0[best] from its owner lane (static register selection)
                T cb = T(0);
#pragma unroll
                for (int k = 0; k < KPL; ++k)
                    if (k == (best >> 5)) cb = c0[k];
                cb = __shfl_sync(SDB_FULL, cb, best & 31);
                n += 1;
                __syncwarp();

                // ---- L L^T x = c0[S] (_kernels.py:129-139); tmp[0..n-2]
                // are unchanged from the previous step, only tmp[n-1] is new.
                {
                    const T* Ln = tri_row(w.L, n - 1);
                    T acc = cb;
                    if (R::kExact || n > 33) {
                        for (int u = 0; u < n - 1; ++u) acc = R::msub(acc, Ln[u], w.tmp[u]);
                    } else {
                        acc -= warp_sum(lane < n - 1 ? Ln[lane] * w.tmp[lane] : T(0));
                    }
                    const T tv = R::div(acc, Ln[n - 1]);
                    __syncwarp();
                    if (lane == 0) w.tmp[n - 1] = tv;
                }
                __syncwarp();
                if (R::kExact || n > 32) {
                    for (int t = n - 1; t >= 0; --t) {
                        T acc = w.tmp[t];
                        for (int u = t + 1; u < n; ++u) acc = R::msub(acc, tri_row(w.L, u)[t], w.x[u]);
                        const T xv = R::div(acc, tri_row(w.L, t)[t]);
                        __syncwarp();
                        if (lane == 0) w.x[t] = xv;
                        __syncwarp();
                    }
                } else {
                    T acc = (lane < n) ? w.tmp[lane] : T(0);
                    T mine = T(0);
                    for (int u = n - 1; u >= 0; --u) {
                        const T xu = R::div(__shfl_sync(SDB_FULL, acc, u), tri_row(w.L, u)[u]);
                        if (lane == u) mine = xu;
                        if (lane < u) acc = R::msub(acc, tri_row(w.L, u)[lane], xu);
                    }
                    __syncwarp();
                    if (lane < n) w.x[lane] = mine;
                    __syncwarp();
                }

                // ---- explicit residual (_kernels.py:141-154)
                T part = T(0);
                for (int r = lane; r < m; r += 32) {
                    T rv = w.y[r];
                    for (int t = 0; t < n; ++t)
                        rv = R::msub(rv, __ldg(Dp + (int64_t)w.ids[t] * m + r), w.x[t]);
                    if constexpr (R::kExact) w.r[r] = rv;
                    else part = fmaf(rv, rv, part);
                }
                T rsq;
                if constexpr (R::kExact) {
                    __syncwarp();
                    rsq = T(0);
                    for (int r = 0; r < m; ++r) rsq = R::mac(rsq, w.r[r], w.r[r]);
                } else {
                    rsq = warp_sum(part);
                }
                rnorm = R::sqrt_(rsq);
                __syncwarp();
                if (rnorm <= eps) break;
            }
        }
        // ---- outputs (selection order; entries >= n zeroed like the reference)
        __syncwarp();
        for (int t = lane; t < cap; t += 32) {
            a.idx[i * cap + t] = (t < n) ? w.ids[t] : 0;
            a.val[i * cap + t] = (t < n) ? w.x[t] : T(0);
        }
        if (lane == 0) {
            a.counts[i] = n;
            a.status[i] = (int8_t)status;
            if (a.rnorm) a.rnorm[i] = rnorm;
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------------------
// FP32 fast path (cap <= 32): same algorithm and stopping rules as k_omp, but
//  * each warp owns a contiguous range of signals and prefetches the next
//    signal's alpha0 row and y into L1 while the current one is coded;
//  * y and the residual live in registers (lane owns rows lane + 32q);
//  * argmax is two redux.sync ops: |corr| >= 0 so its IEEE bits order like
//    the values, and in FP32 the reference's 1e-12 tie window collapses to
//    exact equality (cmax - 1e-12*cmax == cmax), i.e. lowest index among the
//    maxima;
//  * Cholesky / substitutions are lane-parallel column sweeps;
//  * ||r||^2 is tracked through the projection identity ||y||^2 - ||z||^2
//    (z = L^-1 alpha0_S grows by one entry per step); the explicit residual
//    is formed only when
//    that estimate is within 1e-4 ||y||^2 of eps^2 and once for the output;
//  * every load of a step (G[b,b], G[S,b], alpha0[b]) is issued together
//    right after the argmax, so a step costs one L2 round trip;
//  * the support is excluded by overwriting c0[b] with NaN (fmaxf skips it).
// ----------------------------------------------------------------------------
constexpr int FAST_CAP = 32;
constexpr int FAST_TRI = FAST_CAP * (FAST_CAP + 1) / 2;

__host__ __device__ inline int fast_warp_floats(int cap, int m) {
    return FAST_TRI + 4 * FAST_CAP;  // L, 1/diag, tmp, x, ids(as int)
}

// ||y||^2 in FP32 exactly as the fast OMP kernel forms it (lane owns rows
// lane + 32q, fmaf over q, xor-butterfly warp sum), so a precomputed value is
// bitwise the in-kernel one
template <int MPL>
__device__ __forceinline__ float signal_sq(const float* __restrict__ yrow, int lane, int m) {
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < MPL; ++q) {
        const float v = (32 * q + lane < m) ? __ldg(yrow + 32 * q) : 0.0f;
        s = fmaf(v, v, s);
    }
    return warp_sum(s);
}

template <int MPL>
__global__ void __launch_bounds__(256) k_signal_sq(int64_t N, int m, const float* __restrict__ Y, int64_t ldy,
                                                   float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= N) return;
    const float s = signal_sq<MPL>(Y + i * ldy + lane, lane, m);
    if (lane == 0) out[i] = s;
}

int signal_sq_f32(int64_t N, int m, const float* Y, int64_t ldy, float* out, cudaStream_t st) {
    if (N <= 0) return 0;
    const unsigned g = (unsigned)((N + 7) / 8);
    const int mpl = (m + 31) / 32;
    if (mpl <= 1) k_signal_sq<1><<<g, 256, 0, st>>>(N, m, Y, ldy, out);
    else if (mpl <= 2) k_signal_sq<2><<<g, 256, 0, st>>>(N, m, Y, ldy, out);
    else if (mpl <= 5) k_signal_sq<5><<<g, 256, 0, st>>>(N, m, Y, ldy, out);
    else k_signal_sq<8><<<g, 256, 0, st>>>(N, m, Y, ldy, out);
    return (int)cudaGetLastError();
}

// lane owns the KPL consecutive atoms [lane*KPL, lane*KPL + KPL): rows of
// alpha0 and G are read with vector loads when the shape allows it.
template <int KPL>
__device__ __forceinline__ void load_row(float (&v)[KPL], const float* __restrict__ row, int lane,
                                         int K, bool vec) {
    const int j0 = lane * KPL;
    if constexpr (KPL % 4 == 0) {
        if (vec) {
#pragma unroll
            for (int k = 0; k < KPL; k += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(row + j0 + k));
                v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
            }
            return;
        }
    } else if constexpr (KPL % 2 == 0) {
        if (vec) {
#pragma unroll
            for (int k = 0; k < KPL; k += 2) {
                const float2 q = __ldg(reinterpret_cast<const float2*>(row + j0 + k));
                v[k] = q.x; v[k + 1] = q.y;
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < KPL; ++k) v[k] = (j0 + k < K) ? __ldg(row + j0 + k) : 0.0f;
}

// DEFER: code only the signals whose status is -1 (marked by the correlation
// GEMM's step-1 epilogue, sdb_code_step1, for the signals it could not settle);
// each warp scans its contiguous range 32 status bytes at a time (ballot).
template <int KPL, int MPL, bool DEFER>
__global__ void __launch_bounds__(256, (KPL >= 32) ? 2 : (KPL >= 16 ? 3 : (MPL >= 5 ? 3 : 4)))
k_omp_fast(OmpArgs<float> a) {
    extern __shared__ __align__(16) float fsm[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int m = a.m, K = a.K, cap = a.cap;
    float* Ls = fsm + (int64_t)wib * fast_warp_floats(cap, m);
    float* invd = Ls + FAST_TRI;
    float* tmp = invd + FAST_CAP;
    float* xs = tmp + FAST_CAP;
    int* ids = (int*)(xs + FAST_CAP);
    const float eps = a.eps;
    const float eps2 = eps * eps;
    const int j0 = lane * KPL;

    const int64_t gw = (int64_t)blockIdx.x * wpb + wib;
    const int64_t nw = (int64_t)gridDim.x * wpb;
    const int64_t per = (a.N + nw - 1) / nw;
    const int64_t i_begin = gw * per;
    const int64_t i_end = min(a.N, i_begin + per);
    // dynamic: chunks claimed from a.work (always for DEFER; for all signals
    // when the caller supplies the counter — warps then sweep the signals in
    // order, so only a few shards' G matrices are hot in L2 at a time)
    const bool dyn = DEFER || a.work != nullptr;
    if (!dyn && i_begin >= i_end) return;
    const bool vec_a = (K == 32 * KPL) && ((a.lda * 4) % 16 == 0) && (((uintptr_t)a.alpha0 & 15) == 0);
    const bool vec_g = (K == 32 * KPL) && ((K * 4) % 16 == 0) && (((uintptr_t)a.G & 15) == 0);

    // DEFER: the warps claim 32-signal chunks from a device counter (a.work,
    // zeroed by the step-1 launch) — deferred signals cost 2..cap greedy steps,
    // so static ranges would leave the kernel waiting on its unluckiest warp —
    // and code the flagged signals of each chunk (one ballot per chunk); the
    // next claim is issued one chunk ahead so its latency is hidden
    constexpr int CH = 32;   // = warp width: one ballot covers exactly one chunk
    int64_t fc = 0;
    unsigned fl = 0;
    int claim_pending = 0;   // lane 0: result of the claim issued ahead
    auto issue_claim = [&]() {
        if (lane == 0) claim_pending = atomicAdd(a.work, CH);
    };
    auto flags_at = [&](int64_t c) -> unsigned {
        const bool f = (c + lane < a.N) && (!DEFER || __ldg(a.status + c + lane) == (int8_t)-1);
        return __ballot_sync(SDB_FULL, f);
    };
    auto next_flagged = [&]() -> int64_t {
        while (!fl) {
            fc = (int64_t)__shfl_sync(SDB_FULL, claim_pending, 0);
            if (fc >= a.N) return a.N;
            issue_claim();
            fl = flags_at(fc);
        }
        const int64_t r = fc + __ffs(fl) - 1;
        fl &= fl - 1u;
        return r;
    };
    if (dyn) issue_claim();
    const int64_t i_stop = dyn ? a.N : i_end;
    int64_t i = dyn ? next_flagged() : i_begin;
    if (i >= i_stop) return;

    int p = shard_of(a.shard_off, a.P, i);
    int64_t p_end = a.shard_off[p + 1];
    const float* __restrict__ Gp = a.G + (int64_t)p * K * K;
    const float* __restrict__ Dp = a.D + (int64_t)p * K * m;

    // atoms this lane owns that exist (K not a multiple of 32*KPL)
    const int nvalid = max(0, min(KPL, K - j0));
    const bool all_valid = nvalid == KPL;
    const float kNaN = __int_as_float(0x7fffffff);

    for (int64_t i_next; i < i_stop; i = i_next) {
        i_next = dyn ? next_flagged() : i + 1;
        if (i >= p_end) {
            while (i >= p_end) { ++p; p_end = a.shard_off[p + 1]; }
            Gp = a.G + (int64_t)p * K * K;
            Dp = a.D + (int64_t)p * K * m;
        }
        const float* __restrict__ arow = a.alpha0 + i * a.lda;
        int32_t* code_idx = a.idx + i * cap;
        float* code_val = a.val + i * cap;
        const float* __restrict__ yrow = a.Y + i * a.ldy + lane;
        // c0 doubles as the selection mask: a selected (or absent) atom's entry
        // is NaN, which fmaxf skips and whose bits never equal the maximum
        float c0[KPL];
        load_row<KPL>(c0, arow, lane, K, vec_a);
        if (!all_valid) {
#pragma unroll
            for (int k = 0; k < KPL; ++k) c0[k] = (k < nvalid) ? c0[k] : kNaN;
        }
        // the next signal's alpha0 row (and y) are prefetched into L1 (no
        // registers held across the signal, which keeps occupancy at 4 blocks / SM)
        if (i_next < i_stop) {
            const float* an = a.alpha0 + i_next * a.lda;
            if (j0 < K) asm volatile("prefetch.global.L1 [%0];" ::"l"(an + j0));
            if constexpr (KPL > 8) {
                if (j0 + 8 < K) asm volatile("prefetch.global.L1 [%0];" ::"l"(an + j0 + 8));
            }
            if (!a.ysq) {
#pragma unroll
                for (int q = 0; q < MPL; ++q)
                    if (32 * q + lane < m && (lane & 7) == 0)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.Y + i_next * a.ldy + lane + 32 * q));
            }
        }

        // ||y||^2: precomputed (same arithmetic, sdb_signal_sq) or formed here;
        // y itself is only loaded when an explicit residual is needed
        float ysq;
        if (a.ysq) {
            ysq = __ldg(a.ysq + i);
        } else {
            ysq = signal_sq<MPL>(yrow, lane, m);
        }
        float rnorm = 0.0f;  // formed only when reported or needed near the threshold
        float rsq = ysq;
        int n = 0, status = 0;
        // smallest decision margin relative to ||y|| (certification; 1: none close)
        const float ynorm = __fsqrt_rn(ysq);
        float gmin = (a.gap && eps > 0.0f && ynorm > 0.0f) ? fminf(1.0f, fabsf(ynorm - eps) / ynorm) : 1.0f;
        // explicit ||y - D_S x|| (support columns read from L2, independent loads)
        auto resid_norm = [&](int nn) {
            __syncwarp();
            float rr[MPL];
#pragma unroll
            for (int q = 0; q < MPL; ++q) rr[q] = (32 * q + lane < m) ? __ldg(yrow + 32 * q) : 0.0f;
#pragma unroll 4
            for (int t = 0; t < nn; ++t) {
                const float xt = xs[t];
                const float* dc = Dp + ids[t] * m + lane;
#pragma unroll
                for (int q = 0; q < MPL; ++q)
                    if (32 * q + lane < m) rr[q] = fmaf(-__ldg(dc + 32 * q), xt, rr[q]);
            }
            float rs = 0.0f;
#pragma unroll
            for (int q = 0; q < MPL; ++q) rs = fmaf(rr[q], rr[q], rs);
            return __fsqrt_rn(warp_sum(rs));
        };
        if (!(ysq <= eps2 || ysq == 0.0f)) {  // ||y|| <= eps: no atom
            for (int step = 0; step < cap; ++step) {
                // ---- correlations of the residual, support excluded
                float v[KPL];
                if (n == 0) {
#pragma unroll
                    for (int k = 0; k < KPL; ++k) v[k] = fabsf(c0[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < KPL; ++k) v[k] = c0[k];
                    for (int t = 0; t < n; ++t) {
                        float g[KPL];
                        load_row<KPL>(g, Gp + ids[t] * K, lane, K, vec_g);
                        const float coef = xs[t];
#pragma unroll
                        for (int k = 0; k < KPL; ++k) v[k] = fmaf(-g[k], coef, v[k]);
                    }
#pragma unroll
                    for (int k = 0; k < KPL; ++k) v[k] = fabsf(v[k]);
                }
                float lm = 0.0f;
#pragma unroll
                for (int k = 0; k < KPL; ++k) lm = fmaxf(lm, v[k]);
                const uint32_t cbits = __reduce_max_sync(SDB_FULL, __float_as_uint(lm));
                const float cmax = __uint_as_float(cbits);
                if (cmax * cmax <= 1e-26f * rsq) { status = 3; break; }  // cmax <= 1e-13 ||r||
                int cand = 0x7fffffff;
#pragma unroll
                for (int k = KPL - 1; k >= 0; --k)
                    if (__float_as_uint(v[k]) == cbits) cand = j0 + k;
                const int best = (int)__reduce_min_sync(SDB_FULL, (unsigned)cand);
                if (best >= K) { status = 3; break; }  // no candidate (non-finite input)
                if (a.gap && cmax >= 1e-6f * ynorm) {
                    // runner-up |corr| (the best atom excluded)
                    float l2 = 0.0f;
#pragma unroll
                    for (int k = 0; k < KPL; ++k) l2 = (j0 + k == best) ? l2 : fmaxf(l2, v[k]);
                    const float second = __uint_as_float(__reduce_max_sync(SDB_FULL, __float_as_uint(l2)));
                    gmin = fminf(gmin, (cmax - second) / ynorm);
                }

                // ---- every load of this step issued at once: G[b,b], G[S,b], c0[b]
                float dsq = __ldg(Gp + (best * K + best));
                float gacc = (lane < n) ? __ldg(Gp + (ids[lane] * K + best)) : 0.0f;
                const float cb = __ldg(arow + best);
                {
                    const int kk = best - j0;   // in [0, KPL) on the owning lane only
#pragma unroll
                    for (int k = 0; k < KPL; ++k) c0[k] = (kk == k) ? kNaN : c0[k];
                }
                // ---- Cholesky row of the new atom
                float wme = 0.0f;
                if (n > 0) {
                    for (int u = 0; u < n; ++u) {
                        const float wu = __shfl_sync(SDB_FULL, gacc, u) * invd[u];
                        if (lane == u) wme = wu;
                        else if (lane > u && lane < n) gacc = fmaf(-Ls[lane * (lane + 1) / 2 + u], wu, gacc);
                    }
                    dsq -= warp_sum(lane < n ? wme * wme : 0.0f);
                }
                if (dsq <= a.guard) { status = 2; break; }
                const float inv = rsqrtf(dsq);
                const float ldiag = dsq * inv;
                float* Lrow = Ls + n * (n + 1) / 2;
                if (lane < n) Lrow[lane] = wme;
                if (lane == 0) { Lrow[n] = ldiag; invd[n] = inv; ids[n] = best; }
                float tn;
                if (n == 0) {
                    // one atom: tmp = c0[b]/L00, x = tmp/L00
                    tn = cb * inv;
                    if (lane == 0) { tmp[0] = tn; xs[0] = tn * inv; }
                    n = 1;
                } else {
                    tn = (cb - warp_sum(lane < n ? wme * tmp[lane] : 0.0f)) * inv;
                    n += 1;
                    __syncwarp();
                    if (lane == 0) tmp[n - 1] = tn;
                    __syncwarp();
                    float bacc = (lane < n) ? tmp[lane] : 0.0f;
                    float xme = 0.0f;
                    for (int u = n - 1; u >= 0; --u) {
                        const float xu = __shfl_sync(SDB_FULL, bacc, u) * invd[u];
                        if (lane == u) xme = xu;
                        else if (lane < u) bacc = fmaf(-Ls[u * (u + 1) / 2 + lane], xu, bacc);
                    }
                    if (lane < n) xs[lane] = xme;
                }
                // ||r||^2 = ||y||^2 - ||L^-1 c0_S||^2 (projection identity): O(1) per
                // step. Only near the threshold is the explicit residual formed, so
                // the stopping decision is the one the explicit residual gives.
                rsq = fmaxf(fmaf(-tn, tn, rsq), 0.0f);
                __syncwarp();
                if (fabsf(rsq - eps2) <= 1e-4f * ysq) {
                    rnorm = resid_norm(n);
                    if (a.gap) gmin = fminf(gmin, fabsf(rnorm - eps) / ynorm);
                    if (rnorm <= eps) break;
                } else if (rsq <= eps2) {
                    break;
                }
            }
        }
        // reported norm (when requested): explicit residual of the final support
        if (a.rnorm) rnorm = (n > 0) ? resid_norm(n) : __fsqrt_rn(ysq);
        __syncwarp();
        if (lane < cap) {
            code_idx[lane] = (lane < n) ? ids[lane] : 0;
            code_val[lane] = (lane < n) ? xs[lane] : 0.0f;
        }
        if (lane == 0) {
            a.counts[i] = n;
            a.status[i] = (int8_t)status;
            if (a.rnorm) a.rnorm[i] = rnorm;
            if (a.gap) a.gap[i] = gmin;
        }
        __syncwarp();
    }
}

template <int KPL, int MPL>
static int launch_fast_k(const OmpArgs<float>& a, cudaStream_t st) {
    const int wf = fast_warp_floats(a.cap, a.m);
    // 4-warp blocks: register-limited residency of 36 instead of 32 warps per
    // SM (the kernel is bound by per-signal latency chains)
    int wpb = 4;
    while (wpb > 1 && wpb * wf * 4 > 200 * 1024) wpb >>= 1;
    const int smem = wpb * wf * 4;
    auto fn = a.deferred ? k_omp_fast<KPL, MPL, true> : k_omp_fast<KPL, MPL, false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
    }
    // dynamic claiming (a work counter) only pays when every resident warp
    // gets several 32-signal chunks; small batches keep static ranges (one
    // signal per warp when N is below the warp count)
    OmpArgs<float> b = a;
    if (!b.deferred && b.N < (int64_t)32 * 148 * 36) b.work = nullptr;
    const bool dyn = b.deferred || b.work != nullptr;
    const int64_t warps = dyn ? std::min<int64_t>((b.N + 31) / 32, (int64_t)148 * 36)
                              : std::min<int64_t>(b.N, (int64_t)148 * 64);
    const int64_t blocks = (warps + wpb - 1) / wpb;
    fn<<<(unsigned)blocks, wpb * 32, smem, st>>>(b);
    return (int)cudaGetLastError();
}

template <int KPL>
static int launch_fast_m(const OmpArgs<float>& a, cudaStream_t st) {
    const int mpl = (a.m + 31) / 32;
    if (mpl <= 1) return launch_fast_k<KPL, 1>(a, st);
    if (mpl <= 2) return launch_fast_k<KPL, 2>(a, st);
    if (mpl <= 5) return launch_fast_k<KPL, 5>(a, st);
    return launch_fast_k<KPL, 8>(a, st);
}

static int launch_omp_fast(const OmpArgs<float>& a, cudaStream_t st) {
    const int kpl = (a.K + 31) / 32;
    if (kpl <= 1) return launch_fast_m<1>(a, st);
    if (kpl <= 2) return launch_fast_m<2>(a, st);
    if (kpl <= 4) return launch_fast_m<4>(a, st);
    if (kpl <= 8) return launch_fast_m<8>(a, st);
    if (kpl <= 16) return launch_fast_m<16>(a, st);
    if (kpl <= 18) return launch_fast_m<18>(a, st);
    return launch_fast_m<32>(a, st);
}

template <typename T>
int64_t omp_scratch_bytes(int64_t N, int cap, int m, int* use_global) {
    const int64_t wb = omp_warp_bytes<T>(cap, m);
    *use_global = (wb * 8 > 200 * 1024) ? 1 : 0;
    if (!*use_global) return 0;
    const int64_t warps = std::min<int64_t>((N + 0), (int64_t)148 * 32);
    return wb * std::max<int64_t>(warps, 1);
}

template <typename T, int KPL>
static int launch_omp_k(const OmpArgs<T>& a, int blocks, int smem, cudaStream_t st) {
    auto fn = k_omp<T, KPL>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
    }
    fn<<<blocks, 128, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <typename T>
int launch_omp(OmpArgs<T> a, cudaStream_t st) {
    if (a.N <= 0) return 0;
    if constexpr (!Ar<T>::kExact) {
        if (a.cap <= FAST_CAP && a.m <= 256 && a.gscratch == nullptr)
            return launch_omp_fast(a, st);
    }
    const int64_t wb = omp_warp_bytes<T>(a.cap, a.m);
    a.warp_bytes = wb;
    int smem = 0;
    int64_t warps_needed = a.N;
    int64_t blocks;
    // 4-warp blocks: finer residency granularity under the register limit
    // (the exact FP64 kernel holds ~96 registers per thread)
    constexpr int WPB = 4;
    if (a.gscratch) {
        // global scratch holds a.gscratch_warps warps
        blocks = std::max<int64_t>(1, std::min<int64_t>(a.gscratch_warps / WPB, (warps_needed + WPB - 1) / WPB));
    } else {
        smem = (int)(wb * WPB);
        // list mode: the count is only known on the device -- a grid of a few
        // waves strides over it
        blocks = std::min<int64_t>((warps_needed + WPB - 1) / WPB, (int64_t)148 * (a.list ? 16 : 128));
    }
    const int kpl = (a.K + 31) / 32;
    if (kpl <= 1) return launch_omp_k<T, 1>(a, (int)blocks, smem, st);
    if (kpl <= 2) return launch_omp_k<T, 2>(a, (int)blocks, smem, st);
    if (kpl <= 4) return launch_omp_k<T, 4>(a, (int)blocks, smem, st);
    if (kpl <= 8) return launch_omp_k<T, 8>(a, (int)blocks, smem, st);
    if (kpl <= 16) return launch_omp_k<T, 16>(a, (int)blocks, smem, st);
    if (kpl <= 32) return launch_omp_k<T, 32>(a, (int)blocks, smem, st);
    return (int)cudaErrorInvalidValue;  // K > 1024: rejected at the API boundary
}

template int launch_omp<float>(OmpArgs<float>, cudaStream_t);
template int launch_omp<double>(OmpArgs<double>, cudaStream_t);
int64_t omp_warp_bytes_f32(int cap, int m) { return omp_warp_bytes<float>(cap, m); }
int64_t omp_warp_bytes_f64(int cap, int m) { return omp_warp_bytes<double>(cap, m); }

// ----------------------------------------------------------------------------
// CSC packing (sparse_coding.py:294-303): indptr = exclusive scan of counts,
// then each column's entries in ascending atom index.
// ----------------------------------------------------------------------------
constexpr int SCAN_TPB = 256, SCAN_IPT = 8, SCAN_TILE = SCAN_TPB * SCAN_IPT;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* sh, int64_t* total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(SDB_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t s = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(SDB_FULL, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    const int64_t wpre = wid ? sh[wid - 1] : 0;
    *total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return wpre + x - v;
}

__global__ void __launch_bounds__(SCAN_TPB)
k_scan_tiles(const int32_t* __restrict__ counts, int64_t N, int64_t* __restrict__ out,
             int64_t* __restrict__ tile_sums) {
    __shared__ int64_t sh[32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    int64_t loc[SCAN_IPT];
    int64_t s = 0;
#pragma unroll
    for (int q = 0; q < SCAN_IPT; ++q) {
        const int64_t i = base + q;
        loc[q] = s;
        s += (i < N) ? counts[i] : 0;
    }
    int64_t total;
    const int64_t pre = block_exclusive_scan(s, sh, &total);
#pragma unroll
    for (int q = 0; q < SCAN_IPT; ++q) {
        const int64_t i = base + q;
        if (i < N) out[i] = pre + loc[q];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// one block: exclusive scan of the tile sums in chunks with a running carry
__global__ void __launch_bounds__(SCAN_TPB)
k_scan_sums(int64_t* __restrict__ tile_sums, int64_t ntiles, int64_t* __restrict__ grand) {
    __shared__ int64_t sh[32];
    int64_t carry = 0;
    for (int64_t c0 = 0; c0 < ntiles; c0 += SCAN_TPB) {
        const int64_t i = c0 + threadIdx.x;
        const int64_t v = (i < ntiles) ? tile_sums[i] : 0;
        int64_t total;
        const int64_t pre = block_exclusive_scan(v, sh, &total);
        if (i < ntiles) tile_sums[i] = carry + pre;
        carry += total;
    }
    if (threadIdx.x == 0) *grand = carry;
}

__global__ void k_scan_add(int64_t* __restrict__ out, int64_t N, const int64_t* __restrict__ tile_sums) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) out[i] += tile_sums[i / SCAN_TILE];
}

int64_t scan_workspace_bytes(int64_t N) { return sizeof(int64_t) * ((N + SCAN_TILE - 1) / SCAN_TILE + 1); }

// small N (the MOD's P*K bucket counts): one block walks the tiles with a
// running carry — one launch instead of three
__global__ void __launch_bounds__(SCAN_TPB)
k_scan_single(const int32_t* __restrict__ counts, int64_t N, int64_t* __restrict__ out) {
    __shared__ int64_t sh[32];
    int64_t carry = 0;
    for (int64_t t0 = 0; t0 < N; t0 += SCAN_TILE) {
        const int64_t base = t0 + (int64_t)threadIdx.x * SCAN_IPT;
        int64_t loc[SCAN_IPT];
        int64_t s = 0;
#pragma unroll
        for (int q = 0; q < SCAN_IPT; ++q) {
            const int64_t i = base + q;
            loc[q] = s;
            s += (i < N) ? counts[i] : 0;
        }
        int64_t total;
        const int64_t pre = block_exclusive_scan(s, sh, &total);
#pragma unroll
        for (int q = 0; q < SCAN_IPT; ++q) {
            const int64_t i = base + q;
            if (i < N) out[i] = carry + pre + loc[q];
        }
        carry += total;
    }
    if (threadIdx.x == 0) out[N] = carry;
}

// indptr[0..N] (N+1 entries): indptr[0] = 0, indptr[i+1] = sum_{u<=i} counts[u]
int exclusive_scan_counts(const int32_t* counts, int64_t N, int64_t* indptr, int64_t* ws,
                          cudaStream_t st) {
    if (N <= 0) {
        cudaMemsetAsync(indptr, 0, sizeof(int64_t), st);
        return (int)cudaGetLastError();
    }
    const int64_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles <= 8) {
        k_scan_single<<<1, SCAN_TPB, 0, st>>>(counts, N, indptr);
        return (int)cudaGetLastError();
    }
    k_scan_tiles<<<(unsigned)ntiles, SCAN_TPB, 0, st>>>(counts, N, indptr, ws);
    k_scan_sums<<<1, SCAN_TPB, 0, st>>>(ws, ntiles, indptr + N);
    k_scan_add<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(indptr, N, ws);
    return (int)cudaGetLastError();
}

template <typename T>
__global__ void k_pack(int64_t N, int cap, const int32_t* __restrict__ idx, const T* __restrict__ val,
                       const int32_t* __restrict__ counts, const int64_t* __restrict__ indptr,
                       int64_t* __restrict__ out_idx, double* __restrict__ out_val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int n = counts[i];
    const int32_t* ii = idx + i * cap;
    const T* vv = val + i * cap;
    const int64_t b = indptr[i];
    for (int t = 0; t < n; ++t) {
        const int32_t me = ii[t];
        int rank = 0;
        for (int u = 0; u < n; ++u) rank += (ii[u] < me);
        out_idx[b + rank] = me;
        out_val[b + rank] = (double)vv[t];
    }
}

template <typename T>
int pack_csc(int64_t N, int cap, const int32_t* idx, const T* val, const int32_t* counts,
             const int64_t* indptr, int64_t* out_idx, double* out_val, cudaStream_t st) {
    if (N <= 0) return 0;
    k_pack<T><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, cap, idx, val, counts, indptr, out_idx,
                                                           out_val);
    return (int)cudaGetLastError();
}
template int pack_csc<float>(int64_t, int, const int32_t*, const float*, const int32_t*,
                             const int64_t*, int64_t*, double*, cudaStream_t);
template int pack_csc<double>(int64_t, int, const int32_t*, const double*, const int32_t*,
                              const int64_t*, int64_t*, double*, cudaStream_t);

}  // namespace sdb
