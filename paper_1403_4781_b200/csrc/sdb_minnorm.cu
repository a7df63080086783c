// Minimum-norm MOD solve for rank-deficient shards (dictionary_update.py:100:
// D^T = lstsq(X X^T, (Y X^T)^T, rcond=1e-10)).
//
// The batched Cholesky (sdb_chol.cu) flags a shard whose used block has a
// pivot at or below its tolerance (deficient[p] > 0). For those shards only,
// this kernel recomputes A = X X^T and B = Y X^T from the bucketed codes
// (the Cholesky consumed them), diagonalises A with cyclic two-sided Jacobi
// rotations in FP64 (A = Q diag(l) Q^T; A is symmetric positive semidefinite,
// so its singular values are |l|), and forms the minimum-norm solution
//     Z = Q diag(l+) Q^T B,   l+ = 1/l where |l| > rcond * max|l|, else 0,
// which is the pseudo-inverse solution LAPACK's SVD-based lstsq (gelsd)
// returns with the same rank rule. Unused atoms are zero rows of A (exact
// zero eigenvalues), so their rows of Z are zero, as in the reference.
// The shard's rank, deficiency count and an explicit-residual request are
// updated for the MOD finish.
//
// One CTA of 1024 threads per flagged shard (CTAs stride over the shards;
// shards without a flag cost one flag read). Per Jacobi round the K/2
// disjoint pairs of a round-robin tournament rotate at once: one phase forms
// the rotations, the next applies J^T A J to the 2 x 2 blocks of the upper
// triangle (mirrored, so A stays exactly symmetric) and Q J to Q. Sweeps
// repeat until a sweep performs no rotation (|a_pq| <= 1e-16 sqrt(a_pp a_qq)).
// Every sum has a fixed order: the result is deterministic.
#include <algorithm>
#include <cstdint>

#include "sdb_common.cuh"
#include "sdb_mod.h"

namespace sdb {
namespace {

constexpr int MN_THREADS = 1024;
constexpr int MN_MAX_SWEEPS = 40;
constexpr int MN_CTAS = 8;          // flagged shards solved concurrently (one Q slot each)

__device__ __forceinline__ void round_pair(int k, int r, int nn, int& p, int& q) {
    // circle method: position 0 fixed, positions 1..nn-1 rotate by r
    auto who = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + r) % (nn - 1); };
    const int a = who(k), b = who(nn - 1 - k);
    p = min(a, b);
    q = max(a, b);
}

// max_i |A_ii| over the CTA (all threads return it)
__device__ double block_max_diag(const double* A, int K, double* s_red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double mx = 0.0;
    for (int i = tid; i < K; i += MN_THREADS) mx = fmax(mx, fabs(A[(int64_t)i * K + i]));
    mx = warp_max(mx);
    __syncthreads();
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    double v = s_red[lane];
    v = warp_max(v);
    __syncthreads();
    return v;
}

template <typename TY, typename T>
__global__ void __launch_bounds__(MN_THREADS, 1)
k_minnorm(int P, int K, int m, const TY* __restrict__ Y, int64_t ldy, int cap, const int32_t* __restrict__ idx,
          const T* __restrict__ val, const int32_t* __restrict__ counts, const int64_t* __restrict__ bucket_off,
          const int32_t* __restrict__ bent, const int32_t* __restrict__ usage, double rcond,
          double* __restrict__ Aall, double* __restrict__ Ball, int32_t* __restrict__ deficient,
          double* __restrict__ wsq, double* __restrict__ slots) {
    __shared__ double s_c[MN_THREADS / 2 + 1], s_s[MN_THREADS / 2 + 1], s_t[MN_THREADS / 2 + 1];
    __shared__ int s_rot, s_flag;
    __shared__ double s_red[32];
    __shared__ int s_cnt[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = MN_THREADS / 32;
    const int nn = K + (K & 1);   // even number of tournament positions (K odd: one dummy)
    const int np = nn / 2;
    double* Q = slots + (int64_t)blockIdx.x * ((int64_t)K * K + (int64_t)K * m);
    double* Tm = Q + (int64_t)K * K;

    for (int p = blockIdx.x; p < P; p += gridDim.x) {
        if (tid == 0) s_flag = deficient[p];
        __syncthreads();
        if (s_flag == 0) continue;
        double* A = Aall + (int64_t)p * K * K;
        double* B = Ball + (int64_t)p * K * m;
        const int32_t* use = usage + (int64_t)p * K;
        const int64_t* bo = bucket_off + (int64_t)p * K;

        // ---- A = X X^T, B = Y X^T (warp per atom row, bucket entries in order)
        for (int a = warp; a < K; a += nw) {
            double* Ar = A + (int64_t)a * K;
            for (int b = lane; b < K; b += 32) Ar[b] = 0.0;
            __syncwarp();
            double acc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = 0.0;
            if (use[a] > 0) {
                for (int64_t e = bo[a]; e < bo[a + 1]; ++e) {
                    const int64_t f = bent[e];
                    const int64_t i = f / cap;
                    const double xa = (double)val[f];
                    const int n = counts[i];
                    if (lane < n) {
                        const int b = idx[i * cap + lane];
                        Ar[b] += xa * (double)val[i * cap + lane];   // distinct b per lane
                    }
                    __syncwarp();
                    const TY* y = Y + i * ldy;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int c = lane + 32 * k;
                        if (c < m) acc[k] += xa * (double)y[c];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = lane + 32 * k;
                if (c < m) B[(int64_t)a * m + c] = acc[k];
            }
        }
        for (int64_t e = tid; e < (int64_t)K * K; e += MN_THREADS) Q[e] = (e / K == e % K) ? 1.0 : 0.0;
        __syncthreads();
        // absolute floor for rotations (far below anything the rank rule keeps)
        const double floor_abs = 1e-30 * block_max_diag(A, K, s_red);

        // ---- cyclic Jacobi
        for (int sweep = 0; sweep < MN_MAX_SWEEPS; ++sweep) {
            if (tid == 0) s_rot = 0;
            __syncthreads();
            for (int r = 0; r < nn - 1; ++r) {
                for (int k = tid; k < np; k += MN_THREADS) {
                    int pp, qq;
                    round_pair(k, r, nn, pp, qq);
                    double c = 1.0, s = 0.0, t = 0.0;
                    if (qq < K) {
                        const double apq = A[(int64_t)pp * K + qq];
                        const double app = A[(int64_t)pp * K + pp], aqq = A[(int64_t)qq * K + qq];
                        if (fabs(apq) > floor_abs && fabs(apq) > 1e-16 * sqrt(fabs(app) * fabs(aqq))) {
                            const double tau = (aqq - app) / (2.0 * apq);
                            t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                            c = 1.0 / sqrt(1.0 + t * t);
                            s = t * c;
                            atomicAdd(&s_rot, 1);
                        }
                    }
                    s_c[k] = c;
                    s_s[k] = s;
                    s_t[k] = t;
                }
                __syncthreads();
                // J^T A J on the upper-triangle 2x2 blocks (mirrored)
                const int64_t nblk = (int64_t)np * (np + 1) / 2;
                for (int64_t bi = tid; bi < nblk; bi += MN_THREADS) {
                    // bi -> (k, l), k <= l
                    int k = (int)((sqrt(8.0 * (double)bi + 1.0) - 1.0) * 0.5);
                    while ((int64_t)(k + 1) * (k + 2) / 2 <= bi) ++k;
                    while ((int64_t)k * (k + 1) / 2 > bi) --k;
                    const int l = (int)(bi - (int64_t)k * (k + 1) / 2);   // l <= k
                    // rows from pair l, columns from pair k (l <= k)
                    const double c1 = s_c[l], s1 = s_s[l], c2 = s_c[k], s2 = s_s[k];
                    if (s1 == 0.0 && s2 == 0.0) continue;
                    int pr, qr, pc, qc;
                    round_pair(l, r, nn, pr, qr);
                    round_pair(k, r, nn, pc, qc);
                    if (k == l) {
                        if (s1 == 0.0) continue;
                        const double t = s_t[k];
                        const double apq = A[(int64_t)pr * K + qr];
                        A[(int64_t)pr * K + pr] -= t * apq;
                        A[(int64_t)qr * K + qr] += t * apq;
                        A[(int64_t)pr * K + qr] = 0.0;
                        A[(int64_t)qr * K + pr] = 0.0;
                        continue;
                    }
                    const bool vqr = qr < K, vqc = qc < K;
                    const double m00 = A[(int64_t)pr * K + pc];
                    const double m01 = vqc ? A[(int64_t)pr * K + qc] : 0.0;
                    const double m10 = vqr ? A[(int64_t)qr * K + pc] : 0.0;
                    const double m11 = (vqr && vqc) ? A[(int64_t)qr * K + qc] : 0.0;
                    const double r00 = c1 * m00 - s1 * m10, r01 = c1 * m01 - s1 * m11;
                    const double r10 = s1 * m00 + c1 * m10, r11 = s1 * m01 + c1 * m11;
                    const double n00 = c2 * r00 - s2 * r01, n01 = s2 * r00 + c2 * r01;
                    const double n10 = c2 * r10 - s2 * r11, n11 = s2 * r10 + c2 * r11;
                    A[(int64_t)pr * K + pc] = n00;
                    A[(int64_t)pc * K + pr] = n00;
                    if (vqc) { A[(int64_t)pr * K + qc] = n01; A[(int64_t)qc * K + pr] = n01; }
                    if (vqr) { A[(int64_t)qr * K + pc] = n10; A[(int64_t)pc * K + qr] = n10; }
                    if (vqr && vqc) { A[(int64_t)qr * K + qc] = n11; A[(int64_t)qc * K + qr] = n11; }
                }
                // Q J
                for (int64_t e = tid; e < (int64_t)K * np; e += MN_THREADS) {
                    const int i = (int)(e / np), k = (int)(e % np);
                    const double s = s_s[k];
                    if (s == 0.0) continue;
                    const double c = s_c[k];
                    int pp, qq;
                    round_pair(k, r, nn, pp, qq);
                    const double a = Q[(int64_t)i * K + pp], b = Q[(int64_t)i * K + qq];
                    Q[(int64_t)i * K + pp] = c * a - s * b;
                    Q[(int64_t)i * K + qq] = s * a + c * b;
                }
                __syncthreads();
            }
            if (s_rot == 0) break;
            __syncthreads();
        }

        // ---- rank rule and pseudo-inverse weights (diag of A = eigenvalues)
        const double thr = rcond * block_max_diag(A, K, s_red);
        int rk = 0, used = 0;
        for (int i = tid; i < K; i += MN_THREADS) {
            rk += fabs(A[(int64_t)i * K + i]) > thr ? 1 : 0;
            used += use[i] > 0 ? 1 : 0;
        }
        for (int o = 16; o > 0; o >>= 1) {
            rk += __shfl_xor_sync(SDB_FULL, rk, o);
            used += __shfl_xor_sync(SDB_FULL, used, o);
        }
        __syncthreads();
        if (lane == 0) s_cnt[warp] = rk * 2048 + used;
        __syncthreads();
        if (tid == 0) {
            int R = 0, U = 0;
            for (int w = 0; w < nw; ++w) { R += s_cnt[w] / 2048; U += s_cnt[w] % 2048; }
            deficient[p] = U - R;
            wsq[p] = -1.0;   // the Cholesky's ||L^-1 B||^2 no longer applies: explicit residual
        }
        // ---- T = diag(l+) Q^T B, then Z = Q T -> B
        for (int64_t e = tid; e < (int64_t)K * m; e += MN_THREADS) {
            const int i = (int)(e / m), c = (int)(e % m);
            const double li = A[(int64_t)i * K + i];
            double s = 0.0;
            if (fabs(li) > thr) {
                for (int j = 0; j < K; ++j) s += Q[(int64_t)j * K + i] * B[(int64_t)j * m + c];
                s /= li;
            }
            Tm[e] = s;
        }
        __syncthreads();
        for (int64_t e = tid; e < (int64_t)K * m; e += MN_THREADS) {
            const int j = (int)(e / m), c = (int)(e % m);
            double s = 0.0;
            for (int i = 0; i < K; ++i) s += Q[(int64_t)j * K + i] * Tm[(int64_t)i * m + c];
            B[e] = s;
        }
        __syncthreads();
    }
}

}  // namespace

int64_t minnorm_ws_bytes(int P, int m, int K) {
    return (int64_t)std::min(P, MN_CTAS) * ((int64_t)K * K + (int64_t)K * m) * (int64_t)sizeof(double);
}

template <typename TY, typename T>
int minnorm_solve(int P, int K, int m, const TY* Y, int64_t ldy, int cap, const int32_t* idx, const T* val,
                  const int32_t* counts, const int64_t* bucket_off, const int32_t* bent, const int32_t* usage,
                  double rcond, double* A, double* B, int32_t* deficient, double* wsq, double* slots,
                  cudaStream_t st) {
    if (m > 256 || cap > 32) return (int)cudaErrorNotSupported;
    k_minnorm<TY, T><<<std::min(P, MN_CTAS), MN_THREADS, 0, st>>>(P, K, m, Y, ldy, cap, idx, val, counts,
                                                                 bucket_off, bent, usage, rcond, A, B, deficient,
                                                                 wsq, slots);
    return (int)cudaGetLastError();
}
#define SDB_MN_INST(TY, T)                                                                                     \
    template int minnorm_solve<TY, T>(int, int, int, const TY*, int64_t, int, const int32_t*, const T*,       \
                                      const int32_t*, const int64_t*, const int32_t*, const int32_t*, double, \
                                      double*, double*, int32_t*, double*, double*, cudaStream_t);
SDB_MN_INST(float, float)
SDB_MN_INST(double, double)
SDB_MN_INST(float, double)
#undef SDB_MN_INST

}  // namespace sdb
