// FP64 certification of FP32 OMP codes (the "certified FP32" coding mode).
//
// The FP32 / TF32 kernels decide every greedy step with FP32 arithmetic; a
// decision can differ from the reference's FP64 one only when its margin is
// within the FP32 error (~1e-7 ||y||), and the FP32 coefficients carry ~1e-7
// relative error that the MOD step would propagate into the dictionary. This
// pass makes the codes the reference's FP64 codes:
//
//  * signals whose smallest decision margin (gap[i], reported by the FP32
//    kernel: best vs runner-up |corr| and | ||r|| - eps | relative to ||y||)
//    is below `tau`, or whose FP32 status is not OK, are appended to a list
//    and re-coded from scratch by the exact FP64 kernel (k_omp<double>,
//    bitwise the reference's omp_single given the same D, G, y);
//  * every other signal keeps its FP32 support (decided with a margin far
//    above the FP32 error, hence the reference's support) and gets its
//    coefficients refitted in FP64: x = (D_S^T D_S)^-1 D_S^T y with G_SS from
//    the FP64 Gram and D_S^T y from the FP64 dictionary -- the reference's
//    least-squares coefficients on that support (_kernels.py:129-139) to
//    rounding.
//
// Layout: LPS lanes per signal (8 for m <= 64 and cap <= 8: four signals per
// warp; 32 otherwise), lane l holds y[l + LPS v]; the dot products are
// reduced within the lane group. The small SPD solve is a lane-parallel
// right-looking Cholesky (k_certify, group shuffles) or, in the
// dictionary-resident kernel k_certify_sm, one thread per signal after eight
// rounds of dot products (refit_solve_own: the same arithmetic, no shuffles).
// Reads y (4m bytes), the support's dictionary rows (8 m n bytes, shared
// memory or L2) and n(n+1)/2 Gram entries; writes the FP64 code row.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include <type_traits>

#include "sdb_common.cuh"
#include "sdb_internal.h"

namespace sdb {
namespace {

struct CertArgs {
    int64_t N;
    int m, K, cap, P;
    const int64_t* off;
    const float* Y;
    const double* Y64;  // optional: authoritative FP64 rows (same ldy), read instead of Y
    int64_t ldy;
    const double* D;    // P x K x m
    const double* G;    // P x K x K
    const int32_t* idx;
    const int32_t* counts;
    const int8_t* status;
    const float* gap;   // optional
    float tau;
    double* val;        // N x cap (out)
    double* rnorm;      // optional (out)
    int32_t* list;      // fragile signals (out)
    int32_t* nlist;     // count (zeroed by the caller's stream before)
};

template <int LPS>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
    for (int o = LPS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(SDB_FULL, v, o, LPS);
    return v;
}

// 1 / sqrt(g) of a pivot: FP32 seed and two Newton steps in FP64 (to ~1 ulp;
// a dozen instructions on the factorisation's critical path instead of the
// library routine, which still serves pivots outside the FP32 range)
__device__ __forceinline__ double pivot_rsqrt(double g) {
    const float gf = (float)g;
    if (!(gf > 1e-30f && gf < 1e30f)) return rsqrt(g);
    double r = (double)rsqrtf(gf);
    const double h = 0.5 * g;
    r = fma(r, fma(-h * r, r, 0.5), r);
    r = fma(r, fma(-h * r, r, 0.5), r);
    return r;
}

// Sum of part[t] over the 8 lanes of a group, lane t receiving sum t: three
// halving exchanges (4 + 2 + 1 values) instead of eight 3-stage butterflies
__device__ __forceinline__ double gsum8_scatter(const double (&part)[8], int l) {
    double q[4], r[2];
    const bool b2 = l & 4, b1 = l & 2, b0 = l & 1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double send = b2 ? part[j] : part[j + 4];
        const double keep = b2 ? part[j + 4] : part[j];
        q[j] = keep + __shfl_xor_sync(SDB_FULL, send, 4, 8);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const double send = b1 ? q[j] : q[j + 2];
        const double keep = b1 ? q[j + 2] : q[j];
        r[j] = keep + __shfl_xor_sync(SDB_FULL, send, 2, 8);
    }
    const double send = b0 ? r[0] : r[1];
    const double keep = b0 ? r[1] : r[0];
    return keep + __shfl_xor_sync(SDB_FULL, send, 1, 8);
}

// The n x n normal equations of one lane group: lane r holds row r of G_SS
// (columns u <= r) in gr and b_r; returns x_r. Right-looking Cholesky (lane r
// keeps row r: gr[k] -> L[r][k] for k < r; lane k keeps 1 / L[k][k], computed
// once per pivot), forward substitution by broadcasts, back substitution
// through the factor rows staged in shared memory (Ls, per lane group).
template <int LPS>
__device__ __forceinline__ double refit_solve(int n, int nmax, int l, int gbase, double b, double (&gr)[LPS],
                                              double (*Ls)[LPS + 1]) {
    double ik = 1.0;
#pragma unroll
    for (int k = 0; k < LPS; ++k) {
        if (k < nmax) {                                // warp-uniform
            const double gk = __shfl_sync(SDB_FULL, gr[k], gbase + k);   // lane k's pivot
            const double rk = (k < n && gk > 0.0) ? pivot_rsqrt(gk) : 0.0;
            if (l == k) ik = rk;
            if (l > k) gr[k] *= rk;
#pragma unroll
            for (int c = k + 1; c < LPS; ++c) {
                if (c < nmax) {
                    const double lck = __shfl_sync(SDB_FULL, gr[k], gbase + c);   // L[c][k]
                    if (l >= c && l < n) gr[c] = fma(-gr[k], lck, gr[c]);
                }
            }
        }
    }
    // ---- forward L z = b (broadcasts), stage L rows for the back pass
    double z = b;
#pragma unroll
    for (int k = 0; k < LPS; ++k) {
        if (k < nmax) {
            const double zk = __shfl_sync(SDB_FULL, z * ik, gbase + k);   // evaluated on lane k
            if (l == k) z = zk;
            if (l > k) z = fma(-gr[k], zk, z);
        }
    }
    if (l < n) {
#pragma unroll
        for (int u = 0; u < LPS; ++u)
            if (u < nmax) Ls[l][u] = gr[u];
    }
    __syncwarp();
    // ---- back L^T x = z: lane k solves x_k once every x_j, j > k, is in
    double acc = z;
    double x = 0.0;
#pragma unroll
    for (int k = LPS - 1; k >= 0; --k) {
        if (k < nmax) {
            const double xk = __shfl_sync(SDB_FULL, acc * ik, gbase + k);
            if (l == k) x = xk;
            if (l < k && k < n) acc = fma(-Ls[k][l], xk, acc);
        }
    }
    return x;
}

// One lane group of LPS lanes per signal; LPS is also the largest support
// (lane r owns row r of the n x n normal equations). Everything between the
// loads is register-resident: the support Gram row, a lane-parallel right-
// looking Cholesky (columns broadcast by group shuffles), forward substitution
// by broadcasts, back substitution through the factor rows staged in shared
// memory.
template <int LPS, int VPL, int WPB, bool VEC2>
__global__ void __launch_bounds__(WPB * 32, LPS == 8 ? 3 : 1)
k_certify(CertArgs a) {
    constexpr int GPW = 32 / LPS;                      // signals per warp
    __shared__ double sL[WPB * GPW][LPS][LPS + 1];
    __shared__ int64_t s_off[257];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int l = lane & (LPS - 1), g = lane / LPS;
    const int gbase = g * LPS;                         // first lane of the group
    double (*Ls)[LPS + 1] = sL[wib * GPW + g];
    const int m = a.m, K = a.K, cap = a.cap, P = a.P;
    const bool off_smem = P <= 256;

    if (off_smem)
        for (int q = threadIdx.x; q <= P; q += blockDim.x) s_off[q] = a.off[q];
    __syncthreads();
    const int64_t nsig_per_iter = (int64_t)gridDim.x * WPB * GPW;
    // every lane of the warp runs the same number of iterations (group
    // shuffles need the whole warp converged)
    const int64_t iters = (a.N + nsig_per_iter - 1) / nsig_per_iter;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t i = it * nsig_per_iter + ((int64_t)blockIdx.x * WPB + wib) * GPW + g;
        const bool valid = i < a.N;
        int n = valid ? a.counts[i] : 0;
        // supports longer than the lane group (error-bounded coding with a
        // large cap, rare) go to the exact FP64 list as well
        const bool frag = valid && (a.status[i] != 0 || n > LPS || (a.gap != nullptr && !(a.gap[i] >= a.tau)));
        if (frag) {
            if (l == 0) {
                const int pos = atomicAdd(a.nlist, 1);
                a.list[pos] = (int32_t)i;
            }
            n = 0;
        }
        const bool work = valid && !frag;
        int p = 0;
        if (work) {
            int lo = 0, hi = P - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                const int64_t o = off_smem ? s_off[mid] : __ldg(a.off + mid);
                if (o <= i) lo = mid; else hi = mid - 1;
            }
            p = lo;
        }
        const double* Dp = a.D + (int64_t)p * K * m;
        const double* Gp = a.G + (int64_t)p * K * K;
        const int32_t* ids_row = a.idx + (valid ? i : 0) * cap;
        const int my_atom = (l < n) ? ids_row[l] : 0;       // lane r: atom r of the support
        // ---- b = D_S^T y: lane l holds y[l + LPS v]; part[t] for every support atom
        const int nmax0 = __reduce_max_sync(SDB_FULL, n);
        double part[LPS];
#pragma unroll
        for (int t = 0; t < LPS; ++t) part[t] = 0.0;
        int at[LPS];
#pragma unroll
        for (int t = 0; t < LPS; ++t) at[t] = __shfl_sync(SDB_FULL, my_atom, gbase + t);
        if constexpr (VEC2) {
            // lane l: element pairs c = 2l + 2 LPS v (16-byte dictionary loads)
#pragma unroll
            for (int v = 0; v < (VPL + 1) / 2; ++v) {
                const int c = 2 * l + 2 * LPS * v;
                double2 yv = make_double2(0.0, 0.0);
                if (work && c < m) {
                    if (a.Y64) {
                        yv = __ldg(reinterpret_cast<const double2*>(a.Y64 + i * a.ldy + c));
                    } else {
                        const float2 f = __ldg(reinterpret_cast<const float2*>(a.Y + i * a.ldy + c));
                        yv = make_double2((double)f.x, (double)f.y);
                    }
                }
#pragma unroll
                for (int t = 0; t < LPS; ++t) {
                    if (t < nmax0 && t < n && c < m) {
                        const double2 d = __ldg(reinterpret_cast<const double2*>(Dp + (int64_t)at[t] * m + c));
                        part[t] = fma(d.y, yv.y, fma(d.x, yv.x, part[t]));
                    }
                }
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c = l + LPS * v;
                const double yv = (work && c < m) ? (a.Y64 ? __ldg(a.Y64 + i * a.ldy + c)
                                                           : (double)__ldg(a.Y + i * a.ldy + c)) : 0.0;
#pragma unroll
                for (int t = 0; t < LPS; ++t)
                    if (t < nmax0 && t < n && c < m) part[t] = fma(__ldg(Dp + (int64_t)at[t] * m + c), yv, part[t]);
            }
        }
        const int nmax = nmax0;
        double b = 0.0;
#pragma unroll
        for (int t = 0; t < LPS; ++t) {
            if (t < nmax) {                                // warp-uniform
                const double bt = gsum<LPS>(part[t]);
                if (l == t) b = bt;
            }
        }
        // ---- row r of G_SS (columns u <= r), independent loads
        double gr[LPS];
#pragma unroll
        for (int u = 0; u < LPS; ++u)
            gr[u] = (u <= l && l < n) ? __ldg(Gp + (int64_t)my_atom * K + at[u]) : 0.0;
        const double x = refit_solve<LPS>(n, nmax, l, gbase, b, gr, Ls);
        __syncwarp();
        // lane t holds x_t (n <= LPS here); slots past n, including those past
        // LPS when cap > LPS, are zeroed like the reference's
        if (work)
            for (int t = l; t < cap; t += LPS) a.val[i * cap + t] = (t < n) ? x : 0.0;
        if (a.rnorm != nullptr) {
            double rs = 0.0;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c = l + LPS * v;
                double rv = (work && c < m) ? (a.Y64 ? __ldg(a.Y64 + i * a.ldy + c)
                                                     : (double)__ldg(a.Y + i * a.ldy + c)) : 0.0;
#pragma unroll
                for (int t = 0; t < LPS; ++t) {
                    const double xt = __shfl_sync(SDB_FULL, x, gbase + t);
                    if (t < n && c < m) rv = fma(-xt, __ldg(Dp + (int64_t)at[t] * m + c), rv);
                }
                rs = fma(rv, rv, rs);
            }
            rs = gsum<LPS>(rs);
            if (work && l == 0) a.rnorm[i] = sqrt(rs);
        }
        __syncwarp();
    }
}

__device__ __forceinline__ void load_row8i(const int32_t* __restrict__ p, int (&v)[8]) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p)), b = __ldg(reinterpret_cast<const int4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// The n x n normal equations of ONE signal in one thread (n <= 8): G_SS from
// L2 into a packed lower triangle, right-looking Cholesky, forward and back
// substitution, all in registers, no shuffles. The arithmetic is refit_solve's
// operation for operation (same fma operands, same pivot reciprocals), so the
// coefficients are bitwise those of the lane-parallel solve; the diagonal
// slots hold 1 / L[k][k].
__device__ __forceinline__ void refit_solve_own(const double* __restrict__ Gp, int K, const int (&at)[8], int n,
                                                double (&x)[8]) {
    double L[36];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int u = 0; u <= r; ++u)
            L[r * (r + 1) / 2 + u] = (r < n) ? __ldg(Gp + (int64_t)at[r] * K + at[u]) : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k < n) {
            const double gk = L[k * (k + 1) / 2 + k];
            const double rk = gk > 0.0 ? pivot_rsqrt(gk) : 0.0;
            L[k * (k + 1) / 2 + k] = rk;
#pragma unroll
            for (int r = k + 1; r < 8; ++r)
                if (r < n) L[r * (r + 1) / 2 + k] *= rk;
#pragma unroll
            for (int c = k + 1; c < 8; ++c) {
                if (c < n) {
                    const double lck = L[c * (c + 1) / 2 + k];
#pragma unroll
                    for (int r = c; r < 8; ++r)
                        if (r < n) L[r * (r + 1) / 2 + c] = fma(-L[r * (r + 1) / 2 + k], lck, L[r * (r + 1) / 2 + c]);
                }
            }
        }
    }
    // forward L z = b (x holds b on entry)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k < n) {
            x[k] *= L[k * (k + 1) / 2 + k];
#pragma unroll
            for (int r = k + 1; r < 8; ++r)
                if (r < n) x[r] = fma(-L[r * (r + 1) / 2 + k], x[k], x[r]);
        }
    }
    // back L^T x = z
#pragma unroll
    for (int k = 7; k >= 0; --k) {
        if (k < n) {
            x[k] *= L[k * (k + 1) / 2 + k];
#pragma unroll
            for (int r = 0; r < k; ++r) x[r] = fma(-L[k * (k + 1) / 2 + r], x[k], x[r]);
        }
    }
}

// The same refit with the shard's FP64 dictionary resident in shared memory
// (supports of at most 8 atoms, m <= 64): the gathers of the support rows --
// 8 m n bytes per signal, the bulk of k_certify's L2 traffic -- become
// shared-memory reads. A dictionary larger than the budget is taken in two
// column halves (H = 2): pass 0 leaves the partial D_S^T y of every signal in
// its (not yet written) output row, pass 1 adds the other half and solves.
// Work: chunks of CS consecutive signals dealt round-robin to the CTAs (the
// grid stays on a few shards, so the Gram entries come from L2); a chunk is
// cut at shard boundaries and each piece loads its shard's dictionary.
template <int WPB, int CSMAX, bool F64IN>
__global__ void __launch_bounds__(WPB * 32, 1)
k_certify_sm(CertArgs a, int H, int mh, int CS) {
    constexpr int LPS = 8, GPW = 4, NT = WPB * 32, KPT = (CSMAX + NT - 1) / NT;
    static_assert(CSMAX <= 4096, "order entries: 12-bit local index + 3-bit count");
    extern __shared__ __align__(16) unsigned char cs_raw[];
    double* dsm = reinterpret_cast<double*>(cs_raw);                       // K x mh
    // per warp: b = D_S^T y of the 32 signals of eight rounds (9 doubles apart: the
    // owner threads' 8-byte reads are conflict-free)
    double* stage_all = dsm + (size_t)a.K * mh;
    __shared__ uint16_t order[CSMAX];   // the segment's signals by support size: local index | (n - 1) << 12
    __shared__ int hist[LPS + 2];       // signals per support size, then bin offsets; [LPS + 1]: total
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int l = lane & (LPS - 1), g = lane / LPS;
    const int gbase = g * LPS;
    double* stg = stage_all + (size_t)wib * 32 * (LPS + 1);
    const int m = a.m, K = a.K, cap = a.cap, P = a.P;
    const int64_t nchunks = (a.N + CS - 1) / CS;
    const int hp = mh >> 1;                       // double2 per dictionary row half
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t lo = ch * CS, hi = min(a.N, lo + (int64_t)CS);
        int p;
        {
            int blo = 0, bhi = P - 1;
            while (blo < bhi) {
                const int mid = (blo + bhi + 1) >> 1;
                if (__ldg(a.off + mid) <= lo) blo = mid; else bhi = mid - 1;
            }
            p = blo;
        }
        for (int64_t s0 = lo; s0 < hi;) {
            while (__ldg(a.off + p + 1) <= s0) ++p;       // empty shards own no signals
            const int64_t s1 = min(hi, __ldg(a.off + p + 1));
            const double* Dp = a.D + (int64_t)p * K * m;
            const double* Gp = a.G + (int64_t)p * K * K;
            // ---- order the segment's signals by support size, so the four
            // signals of a warp share their loop bounds (error-bounded coding
            // mixes supports of 1 and of 8 atoms). Fragile signals go to the
            // list, empty supports are zero-filled here; the order within a size
            // is arbitrary (every signal's result is independent of it)
            __syncthreads();                              // the previous segment's order is no longer read
            if (threadIdx.x < LPS + 2) hist[threadIdx.x] = 0;
            __syncthreads();
            int keys[KPT];
#pragma unroll
            for (int q = 0; q < KPT; ++q) {
                const int li = threadIdx.x + q * NT;
                keys[q] = -1;
                if (li < CS && s0 + li < s1) {
                    const int64_t i = s0 + li;
                    const int n = __ldg(a.counts + i);
                    const bool frag = __ldg(a.status + i) != 0 || n > LPS ||
                                      (a.gap != nullptr && !(__ldg(a.gap + i) >= a.tau));
                    if (frag) {
                        const int pos = atomicAdd(a.nlist, 1);
                        a.list[pos] = (int32_t)i;
                    } else if (n == 0) {
                        for (int t = 0; t < cap; ++t) a.val[i * cap + t] = 0.0;
                    } else {
                        keys[q] = (n << 16) | atomicAdd(&hist[n], 1);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int run = 0;
                for (int n = 1; n <= LPS; ++n) {
                    const int c = hist[n];
                    hist[n] = run;
                    run += c;
                }
                hist[LPS + 1] = run;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < KPT; ++q) {
                if (keys[q] >= 0) {
                    const int n = keys[q] >> 16;
                    order[hist[n] + (keys[q] & 0xffff)] = (uint16_t)((threadIdx.x + q * NT) | ((n - 1) << 12));
                }
            }
            const int total = hist[LPS + 1];
            for (int h = 0; h < H; ++h) {
                const int c0 = h * mh;
                __syncthreads();                          // the previous rows are no longer read; order[] is complete
                for (int e = threadIdx.x; e < K * hp; e += NT) {
                    const int j = e / hp, c = c0 + 2 * (e - j * hp);
                    double2 v = make_double2(0.0, 0.0);
                    if (c < m) v = __ldg(reinterpret_cast<const double2*>(Dp + (int64_t)j * m + c));
                    reinterpret_cast<double2*>(dsm)[e] = v;
                }
                __syncthreads();
                const bool last = h == H - 1;
                // lane l's atom, the signal values of this column range and (pass 1)
                // the partial sum are requested one iteration ahead of their use
                struct Pre {
                    int64_t i;
                    int n, atom;
                    // FP32 rows stay raw until their use (a conversion here would wait
                    // for the load one round early)
                    typename std::conditional<F64IN, double2, float2>::type y[4];
                    double bp;
                };
                auto fetch = [&](int w) {
                    Pre f;
                    f.i = 0; f.n = 0; f.atom = 0; f.bp = 0.0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) { f.y[v].x = 0; f.y[v].y = 0; }
                    if (w < total) {
                        const int o = order[w];
                        const int64_t i = s0 + (o & 0xfff);
                        f.i = i;
                        f.n = (o >> 12) + 1;
                        if (l < cap) f.atom = __ldg(a.idx + i * cap + l);
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int cl = 2 * l + 2 * LPS * v, c = c0 + cl;
                            if (cl < mh && c < m) {
                                if constexpr (F64IN) {
                                    f.y[v] = __ldg(reinterpret_cast<const double2*>(a.Y64 + i * a.ldy + c));
                                } else {
                                    f.y[v] = __ldg(reinterpret_cast<const float2*>(a.Y + i * a.ldy + c));
                                }
                            }
                        }
                        if (last && H > 1 && l < cap) f.bp = a.val[i * cap + l];
                    }
                    return f;
                };
                Pre nxt = fetch(wib * GPW + g);
                for (int base = 0; base < total; base += WPB * GPW) {
                    const int w = base + wib * GPW + g;
                    const bool work = w < total;
                    const Pre cur = nxt;
                    nxt = fetch(w + WPB * GPW);
                    const int64_t i = cur.i;
                    const int n = cur.n;
                    const int my_atom = (l < n) ? cur.atom : 0;
                    const int nmax = __reduce_max_sync(SDB_FULL, n);
                    int at[LPS];
#pragma unroll
                    for (int t = 0; t < LPS; ++t) at[t] = __shfl_sync(SDB_FULL, my_atom, gbase + t);
                    // ---- this column range's share of b = D_S^T y (lane l: pairs 2l + 16v)
                    double part[LPS];
#pragma unroll
                    for (int t = 0; t < LPS; ++t) part[t] = 0.0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int cl = 2 * l + 2 * LPS * v;       // column within the range
                        if (cl < mh) {                            // uniform in v
                            const double yx = (double)cur.y[v].x, yy = (double)cur.y[v].y;
#pragma unroll
                            for (int t = 0; t < LPS; ++t) {
                                if (t < nmax && t < n) {
                                    const double2 d = *reinterpret_cast<const double2*>(dsm + (size_t)at[t] * mh + cl);
                                    part[t] = fma(d.y, yy, fma(d.x, yx, part[t]));
                                }
                            }
                        }
                    }
                    // lane t of the group: b_t (single-atom rounds, warp-uniform: one
                    // butterfly, the same additions)
                    double b;
                    if (nmax <= 1) {
                        b = gsum<LPS>(part[0]);
                        if (l != 0) b = 0.0;
                    } else {
                        b = gsum8_scatter(part, l);
                    }
                    if (!last) {
                        // partial sums wait in the signal's output row
                        if (work && l < cap) a.val[i * cap + l] = b;
                        continue;
                    }
                    b += cur.bp;
                    // ---- eight rounds fill the warp's stage (round k, group g ->
                    // slot 4k + g); then thread 4k + g solves that signal's normal
                    // equations on its own
                    const int rnd = (base / (WPB * GPW)) & 7;
                    if (work) stg[(rnd * GPW + g) * (LPS + 1) + l] = b;
                    if (rnd == 7 || base + WPB * GPW >= total) {
                        __syncwarp();
                        const int w_own = base - rnd * (WPB * GPW) + (lane >> 2) * (WPB * GPW) + wib * GPW + (lane & 3);
                        if ((lane >> 2) <= rnd && w_own < total) {
                            const int o = order[w_own];
                            const int64_t io = s0 + (o & 0xfff);
                            const int no = (o >> 12) + 1;
                            int at[8];
#pragma unroll
                            for (int t = 0; t < 8; ++t) at[t] = 0;
                            if (cap == 8) {
                                load_row8i(a.idx + io * 8, at);
                            } else {
#pragma unroll
                                for (int t = 0; t < 8; ++t)
                                    if (t < cap) at[t] = __ldg(a.idx + io * cap + t);
                            }
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                if (t >= no) at[t] = 0;
                            double x[8];
#pragma unroll
                            for (int t = 0; t < 8; ++t) x[t] = stg[lane * (LPS + 1) + t];
                            refit_solve_own(Gp, K, at, no, x);
                            if (cap == 8) {
                                double2* o2 = reinterpret_cast<double2*>(a.val + io * 8);
#pragma unroll
                                for (int t = 0; t < 8; t += 2)
                                    o2[t >> 1] = make_double2(t < no ? x[t] : 0.0, t + 1 < no ? x[t + 1] : 0.0);
                            } else {
#pragma unroll
                                for (int t = 0; t < 8; ++t)
                                    if (t < cap) a.val[io * cap + t] = (t < no) ? x[t] : 0.0;
                            }
                        }
                        __syncwarp();
                    }
                }
            }
            s0 = s1;
        }
    }
}

template <int LPS, int VPL, int WPB>
int launch_cert(const CertArgs& a, cudaStream_t st) {
    constexpr int GPW = 32 / LPS;
    const int64_t per = (int64_t)WPB * GPW;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((a.N + per - 1) / per, 148 * 64 / WPB));
    // 16-byte loads when every row starts 16-byte aligned
    const bool vec2 = (a.m % 2 == 0) && (a.ldy % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.D) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(a.Y64 ? (const void*)a.Y64 : (const void*)a.Y) & 15) == 0);
    if (vec2) k_certify<LPS, VPL, WPB, true><<<(unsigned)blocks, WPB * 32, 0, st>>>(a);
    else k_certify<LPS, VPL, WPB, false><<<(unsigned)blocks, WPB * 32, 0, st>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace

int certify_refit(int64_t N, int m, int K, int cap, int P, const int64_t* off, const float* Y, const double* Y64,
                  int64_t ldy, const double* D, const double* G, const int32_t* idx, const int32_t* counts,
                  const int8_t* status, const float* gap, float tau, double* val, double* rnorm, int32_t* list,
                  int32_t* nlist, bool short_supports, cudaStream_t st) {
    if (N <= 0) return 0;
    CertArgs a{N, m, K, cap, P, off, Y, Y64, ldy, D, G, idx, counts, status, gap, tau, val, rnorm, list, nlist};
    // 8-lane groups whenever the supports are short (cap <= 8, or error-
    // bounded coding: the few longer supports are re-coded exactly)
    if ((cap <= 8 || short_supports) && m <= 64) {
        // dictionary-resident variant: 16-byte aligned rows, shards long enough
        // to amortise the dictionary loads, no residual norms
        static const bool sm_off = getenv("SDB_CERT_SM") != nullptr && atoi(getenv("SDB_CERT_SM")) == 0;
        constexpr int WPB = 16;
        const bool vec2 = (m % 2 == 0) && (ldy % 4 == 0) && ((reinterpret_cast<uintptr_t>(D) & 15) == 0) &&
                          ((reinterpret_cast<uintptr_t>(Y64 ? (const void*)Y64 : (const void*)Y) & 15) == 0);
        const int64_t budget = 160 * 1024;
        int H = 1, mh = (m + 1) / 2 * 2;
        if ((int64_t)K * mh * 8 > budget) {
            H = 2;
            mh = ((m + 1) / 2 + 15) / 16 * 16;
        }
        const int64_t dyn = (int64_t)K * mh * 8 + (int64_t)WPB * 4 * 8 * 9 * 8;
        if (!sm_off && vec2 && rnorm == nullptr && N >= (int64_t)P * 1024 && (int64_t)K * mh * 8 <= budget &&
            mh <= 64) {
            constexpr int CSMAX = 4096;
            int dev = 0, n_sm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
            // chunks: the same number per CTA, whole lane-group rounds, at most
            // CSMAX signals; short chunks would not amortise the dictionary
            // loads -> the gather kernel
            const int64_t rounds = ((N + n_sm - 1) / n_sm + CSMAX - 1) / CSMAX;     // chunks per CTA
            const int64_t per = (N + n_sm * rounds - 1) / (n_sm * rounds);
            const int CS = (int)std::min<int64_t>(CSMAX, (per + WPB * 4 - 1) / (WPB * 4) * (WPB * 4));
            if (CS < 480) return launch_cert<8, 8, 8>(a, st);
            const int64_t nchunks = (N + CS - 1) / CS;
            const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(n_sm, nchunks));
            if (Y64 != nullptr) {
                cudaError_t e = set_max_smem((const void*)k_certify_sm<WPB, CSMAX, true>, (int)dyn);
                if (e != cudaSuccess) return (int)e;
                k_certify_sm<WPB, CSMAX, true><<<grid, WPB * 32, dyn, st>>>(a, H, mh, CS);
            } else {
                cudaError_t e = set_max_smem((const void*)k_certify_sm<WPB, CSMAX, false>, (int)dyn);
                if (e != cudaSuccess) return (int)e;
                k_certify_sm<WPB, CSMAX, false><<<grid, WPB * 32, dyn, st>>>(a, H, mh, CS);
            }
            return (int)cudaGetLastError();
        }
        return launch_cert<8, 8, 8>(a, st);
    }
    if ((cap <= 8 || short_supports) && m <= 256) return launch_cert<8, 32, 8>(a, st);
    if (cap <= 16 && m <= 64) return launch_cert<16, 4, 8>(a, st);
    if (cap <= 16 && m <= 256) return launch_cert<16, 16, 4>(a, st);
    if (cap <= 32 && m <= 64) return launch_cert<32, 2, 4>(a, st);
    if (cap <= 32 && m <= 128) return launch_cert<32, 4, 4>(a, st);
    if (cap <= 32 && m <= 256) return launch_cert<32, 8, 4>(a, st);
    return (int)cudaErrorNotSupported;
}

}  // namespace sdb
