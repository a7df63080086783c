// Shard-batched FP64 blocked Cholesky solve of the MOD normal equations
// A Z = B (A = X X^T, K x K; B = (Y X^T)^T, K x m), replacing
// numpy.linalg.lstsq in dictionary_update.py:100.
//
// Right-looking, 64-wide panels; every launch covers all P shards:
//   prep        mask unused atoms (identity rows/cols), pivot tolerance
//   per panel j: diag   A_jj = L_jj L_jj^T (one CTA: two warp-synchronous
//                       32-wide sub-blocks + a shuffle row sweep)
//                panel  L_ij = A_ij L_jj^-T (i > j, row sweeps), W_j = L_jj^-1 B_j
//                update A_ik -= L_ij L_kj^T (lower tiles), B_i -= L_ij W_j
//   per panel j (descending): Z_j = L_jj^-T W_j ; W_i -= L_ji^T Z_j (i < j)
// Numerically dependent pivots (<= rcond * max used diagonal) drop their atom
// (zero column of L, zero solution row), which the caller treats as dead.
#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_chol.h"

#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

namespace sdb {

constexpr int CB = 64;       // panel / tile width
constexpr int CBP = CB + 1;  // padded smem row (tile GEMMs: 16 consecutive rows per warp)
// row stride for the sweep kernels: a warp touches 8 rows x 4 columns; stride
// 68 doubles (== 4 mod 16 bank pairs) spreads them over all 16 pairs twice
constexpr int CBD = 68;

__global__ void __launch_bounds__(256)
k_chol_prep(int K, double* __restrict__ Aall, const int32_t* __restrict__ usage,
            double rel_tol, double* __restrict__ tol_out, int32_t* __restrict__ ndep) {
    const int p = blockIdx.y;
    double* A = Aall + (int64_t)p * K * K;
    const int32_t* use = usage + (int64_t)p * K;
    const int64_t KK = (int64_t)K * K;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < KK;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / K), c = (int)(e % K);
        if (!use[r] || !use[c]) A[e] = (r == c) ? 1.0 : 0.0;
    }
    if (blockIdx.x == 0) {
        __shared__ double sh[256];
        double mx = 0.0;
        for (int r = threadIdx.x; r < K; r += 256)
            if (use[r]) mx = fmax(mx, A[(int64_t)r * K + r]);
        sh[threadIdx.x] = mx;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            tol_out[p] = rel_tol * sh[0];
            ndep[p] = 0;
        }
    }
}

// ---- row sweep X L^T = A for rows of Xs (4 lanes per row, 8 rows per warp):
// x_c = (a_c - sum_{q<c} x_q L[c][q]) / L[c][c], written in place into Xs.
template <int S>
__device__ __forceinline__ void rows_trsm(double (*Xs)[S], int nrows, double (*Ls)[S],
                                          const double* inv, const int8_t* sdep, int nb) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane & 3;
    const int r = warp * 8 + (lane >> 2);
    for (int c = 0; c < nb; ++c) {
        double v = 0.0;
        if (r < nrows)
            for (int q = h; q < c; q += 4) v = fma(Xs[r][q], Ls[c][q], v);
        v += __shfl_xor_sync(SDB_FULL, v, 1);
        v += __shfl_xor_sync(SDB_FULL, v, 2);
        if (r < nrows && h == 0) Xs[r][c] = sdep[c] ? 0.0 : (Xs[r][c] - v) * inv[c];
        __syncwarp();
    }
}

// ---- substitution on a 64-column tile W (smem, W[row][col]): column t is
// handled by the 4 lanes 4t..4t+3 of one warp (8 columns per warp), each
// summing a quarter of the dot product, combined by shuffles. lower: solve
// L w = b (forward, dependent rows -> 0); !lower: solve L^T z = w (backward).
template <int S>
__device__ __forceinline__ void cols_trsv(double (*W)[S], int ncols, double (*Ls)[S],
                                          const double* inv, const int8_t* sdep, int nb,
                                          bool lower) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane & 3;
    const int t = warp * 8 + (lane >> 2);
    const bool act = t < ncols;
    for (int k = 0; k < nb; ++k) {
        const int rr = lower ? k : nb - 1 - k;
        double v = 0.0;
        if (act) {
            if (lower) {
                for (int q = h; q < rr; q += 4) v = fma(Ls[rr][q], W[q][t], v);
            } else {
                for (int q = rr + 1 + h; q < nb; q += 4) v = fma(Ls[q][rr], W[q][t], v);
            }
        }
        v += __shfl_xor_sync(SDB_FULL, v, 1);
        v += __shfl_xor_sync(SDB_FULL, v, 2);
        if (act && h == 0) {
            const double nv = (W[rr][t] - v) * inv[rr];
            W[rr][t] = (lower && sdep[rr]) ? 0.0 : nv;
        }
        __syncwarp();
    }
}

// factor the diagonal block of panel j0, right-looking, register resident:
// thread t owns row r = t/4 and its 16 columns q = 4j + t%4 in registers for
// the whole factorisation (the 64-column loop is unrolled so every register
// index is static). Per column: the pivot owner publishes the pivot, the
// column's owners publish the scaled column through a double-buffered smem
// vector, every thread updates its 16 values — two CTA barriers per column.
__global__ void __launch_bounds__(256)
k_chol_diag(int K, int j0, double* __restrict__ Aall, double* __restrict__ Tall,
            const double* __restrict__ tol, int8_t* __restrict__ depmask, int32_t* __restrict__ ndep) {
    extern __shared__ double dsm[];
    double (*Ls)[CBP] = reinterpret_cast<double (*)[CBP]>(dsm);
    double (*Ts)[CBP] = reinterpret_cast<double (*)[CBP]>(dsm + CB * CBP);
    double (*Ms)[33] = reinterpret_cast<double (*)[33]>(dsm + 2 * CB * CBP);
    __shared__ double colv[2][CB];
    __shared__ double s_inv[2];
    __shared__ int8_t sdep[CB];
    const int p = blockIdx.x;
    double* A = Aall + (int64_t)p * K * K;
    const int nb = min(CB, K - j0);
    const int tid = threadIdx.x;
    const int r = tid >> 2, g = tid & 3;
    double v[CB / 4];
    {
        const double* arow = A + (int64_t)(j0 + r) * K + j0;
#pragma unroll
        for (int j = 0; j < CB / 4; ++j) {
            const int q = 4 * j + g;
            v[j] = (r < nb && q <= r) ? arow[q] : 0.0;
        }
    }
    const double tl = tol[p];
#pragma unroll
    for (int c = 0; c < CB; ++c) {
        if (c < nb) {
            const int buf = c & 1;
            const int jc = c >> 2;
            if (r == c && g == (c & 3)) {  // pivot owner
                const double d = v[jc];
                const bool dep = !(d > tl);
                double y = (double)rsqrtf((float)d);
                y = y * fma(-0.5 * d * y, y, 1.5);
                y = y * fma(-0.5 * d * y, y, 1.5);
                v[jc] = dep ? 1.0 : d * y;
                sdep[c] = dep ? 1 : 0;
                s_inv[buf] = dep ? 0.0 : y;
            }
            __syncthreads();
            if (r > c && r < nb && g == (c & 3)) {
                v[jc] *= s_inv[buf];
                colv[buf][r] = v[jc];
            }
            __syncthreads();
            if (r > c && r < nb) {
                const double lr = colv[buf][r];
#pragma unroll
                for (int j = 0; j < CB / 4; ++j) {
                    const int q = 4 * j + g;
                    if (q > c && q <= r) v[j] = fma(-lr, colv[buf][q], v[j]);
                }
            }
        }
    }
    {
        double* arow = A + (int64_t)(j0 + r) * K + j0;
#pragma unroll
        for (int j = 0; j < CB / 4; ++j) {
            const int q = 4 * j + g;
            if (r < nb && q <= r) arow[q] = v[j];
            Ls[r][q] = (r < nb && q <= r) ? v[j] : 0.0;
        }
    }
    __syncthreads();
    // T = L^-1 (64x64 lower), blocked 2x2 of 32: warps 0/1 invert the diagonal
    // sub-blocks column-parallel, then T21 = -T22 L21 T11 by two tile GEMMs.
    // Dependent atoms get a zero row and column in T.
    {
        const int lane = tid & 31, warp = tid >> 5;
        if (warp < 2) {
            const int o = warp * 32, c = o + lane;
            for (int rr2 = 0; rr2 < 32; ++rr2) Ts[o + rr2][c] = 0.0;
            if (c < nb && !sdep[c]) {
                Ts[c][c] = 1.0 / Ls[c][c];
                for (int rr2 = c + 1; rr2 < min(o + 32, nb); ++rr2) {
                    double acc = 0.0;
                    for (int q = c; q < rr2; ++q) acc = fma(Ls[rr2][q], Ts[q][c], acc);
                    Ts[rr2][c] = sdep[rr2] ? 0.0 : -acc / Ls[rr2][rr2];
                }
            }
        }
        // zero the upper-right block
        for (int e = tid; e < 32 * 32; e += 256) Ts[e >> 5][32 + (e & 31)] = 0.0;
        __syncthreads();
        // M = L21 T11 (32x32), then T21 = -T22 M
        for (int e = tid; e < 32 * 32; e += 256) {
            const int rr2 = e >> 5, c = e & 31;
            double acc = 0.0;
            for (int q = c; q < 32; ++q) acc = fma(Ls[32 + rr2][q], Ts[q][c], acc);
            Ms[rr2][c] = acc;
        }
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += 256) {
            const int rr2 = e >> 5, c = e & 31;
            double acc = 0.0;
            for (int q = 0; q <= rr2; ++q) acc = fma(Ts[32 + rr2][32 + q], Ms[q][c], acc);
            Ts[32 + rr2][c] = -acc;
        }
        __syncthreads();
        double* T = Tall + ((int64_t)p * ((K + CB - 1) / CB) + j0 / CB) * CB * CB;
        for (int e = tid; e < CB * CB; e += 256) T[e] = Ts[e / CB][e % CB];
    }
    if (tid < nb) depmask[(int64_t)p * K + j0 + tid] = sdep[tid];
    if (tid == 0) {
        int nd = 0;
        for (int c = 0; c < nb; ++c) nd += sdep[c];
        ndep[p] += nd;
    }
}

// 64x64 tile update  C -= X Y^T  with X (64 x nb), Y (64 x nb) from smem;
// each thread owns a 4x4 micro-tile (rows ty+16a, cols tx+16b).
__device__ __forceinline__ void tile_update(double (*Xs)[CBP], double (*Ys)[CBP], int nb,
                                            double acc[4][4]) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int q = 0; q < nb; ++q) {
        double xv[4], yv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = Xs[ty + 16 * a][q];
#pragma unroll
        for (int b = 0; b < 4; ++b) yv[b] = Ys[tx + 16 * b][q];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(xv[a], yv[b], acc[a][b]);
    }
}

// blockIdx.x == 0: W_j = T_j B_j (the panel's right-hand-side rows)
// blockIdx.x >= 1: 64-row block of the panel, L_ij = A_ij T_j^T
// both as register-blocked 64x64 tile GEMMs (T_j = L_jj^-1 from k_chol_diag)
__global__ void __launch_bounds__(256)
k_chol_panel(int K, int m, int j0, double* __restrict__ Aall, double* __restrict__ Ball,
             const double* __restrict__ Tall) {
    extern __shared__ double csm[];
    double (*Xs)[CBP] = reinterpret_cast<double (*)[CBP]>(csm);
    double (*Ys)[CBP] = reinterpret_cast<double (*)[CBP]>(csm + CB * CBP);
    const int p = blockIdx.y;
    const int nb = min(CB, K - j0);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const double* T = Tall + ((int64_t)p * ((K + CB - 1) / CB) + j0 / CB) * CB * CB;
    double acc[4][4];
    if (blockIdx.x == 0) {
        double* B = Ball + (int64_t)p * K * m + (int64_t)j0 * m;
        for (int e = tid; e < CB * CB; e += 256) Xs[e / CB][e % CB] = T[e];  // Xs[r][q] = T[r][q]
        for (int c0 = 0; c0 < m; c0 += CB) {
            const int nc = min(CB, m - c0);
            __syncthreads();
            for (int e = tid; e < CB * CB; e += 256) {  // Ys[col][q] = B[q][col]
                const int q = e / CB, c = e % CB;
                Ys[c][q] = (q < nb && c < nc) ? B[(int64_t)q * m + c0 + c] : 0.0;
            }
            __syncthreads();
            tile_update(Xs, Ys, nb, acc);
#pragma unroll
            for (int a2 = 0; a2 < 4; ++a2) {
                const int r = ty + 16 * a2;
#pragma unroll
                for (int b2 = 0; b2 < 4; ++b2) {
                    const int c = tx + 16 * b2;
                    if (r < nb && c < nc) B[(int64_t)r * m + c0 + c] = acc[a2][b2];
                }
            }
        }
        return;
    }
    const int i0 = j0 + nb + (blockIdx.x - 1) * CB;
    if (i0 >= K) return;
    const int ni = min(CB, K - i0);
    double* A = Aall + (int64_t)p * K * K;
    for (int e = tid; e < CB * CB; e += 256) {
        const int r = e / CB, c = e % CB;
        Xs[r][c] = (r < ni && c < nb) ? A[(int64_t)(i0 + r) * K + j0 + c] : 0.0;
        Ys[r][c] = T[e];  // Ys[c][q] = T[c][q]  ->  out[r][c] = sum_q X[r][q] T[c][q]
    }
    __syncthreads();
    tile_update(Xs, Ys, nb, acc);
#pragma unroll
    for (int a2 = 0; a2 < 4; ++a2) {
        const int r = ty + 16 * a2;
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
            const int c = tx + 16 * b2;
            if (r < ni && c < nb) A[(int64_t)(i0 + r) * K + j0 + c] = acc[a2][b2];
        }
    }
}

// trailing update: blockIdx.x enumerates lower tiles (I >= J) of the trailing
// matrix, then RHS tiles (I, column chunk).
__global__ void __launch_bounds__(256)
k_chol_update(int K, int m, int j0, double* __restrict__ Aall, double* __restrict__ Ball) {
    extern __shared__ double csm[];
    double (*Xs)[CBP] = reinterpret_cast<double (*)[CBP]>(csm);
    double (*Ys)[CBP] = reinterpret_cast<double (*)[CBP]>(csm + CB * CBP);
    const int p = blockIdx.y;
    const int nb = min(CB, K - j0);
    const int t0 = j0 + nb;
    const int nt = (K - t0 + CB - 1) / CB;
    const int ntri = nt * (nt + 1) / 2;
    const int nmc = (m + CB - 1) / CB;
    int tile = blockIdx.x;
    if (tile >= ntri + nt * nmc) return;
    double* A = Aall + (int64_t)p * K * K;
    double* B = Ball + (int64_t)p * K * m;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    if (tile < ntri) {
        int bi = 0;
        while ((bi + 1) * (bi + 2) / 2 <= tile) ++bi;
        const int bj = tile - bi * (bi + 1) / 2;
        const int r0 = t0 + bi * CB, c0 = t0 + bj * CB;
        for (int e = tid; e < CB * CB; e += 256) {
            const int r = e / CB, q = e % CB;
            Xs[r][q] = (r0 + r < K && q < nb) ? A[(int64_t)(r0 + r) * K + j0 + q] : 0.0;
            Ys[r][q] = (c0 + r < K && q < nb) ? A[(int64_t)(c0 + r) * K + j0 + q] : 0.0;
        }
        __syncthreads();
        double acc[4][4];
        tile_update(Xs, Ys, nb, acc);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int gr = r0 + ty + 16 * a;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int gc = c0 + tx + 16 * b;
                if (gr < K && gc <= gr) A[(int64_t)gr * K + gc] -= acc[a][b];
            }
        }
        return;
    }
    tile -= ntri;
    const int bi = tile / nmc, mc = tile % nmc;
    const int r0 = t0 + bi * CB, c0 = mc * CB;
    // C[r][c] (B rows r0.., cols c0..) -= sum_q L[r0+r][j0+q] * W[j0+q][c0+c]
    for (int e = tid; e < CB * CB; e += 256) {
        const int r = e / CB, q = e % CB;
        Xs[r][q] = (r0 + r < K && q < nb) ? A[(int64_t)(r0 + r) * K + j0 + q] : 0.0;
        const int qq = e / CB, c = e % CB;  // coalesced over c
        Ys[c][qq] = (qq < nb && c0 + c < m) ? B[(int64_t)(j0 + qq) * m + c0 + c] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
    tile_update(Xs, Ys, nb, acc);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int gr = r0 + ty + 16 * a;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int gc = c0 + tx + 16 * b;
            if (gr < K && gc < m) B[(int64_t)gr * m + gc] -= acc[a][b];
        }
    }
}

// back substitution, panel j0: Z_j = T_j^T W_j in place (tile GEMM)
__global__ void __launch_bounds__(256)
k_back_diag(int K, int m, int j0, const double* __restrict__ Tall, double* __restrict__ Ball) {
    extern __shared__ double csm[];
    double (*Xs)[CBP] = reinterpret_cast<double (*)[CBP]>(csm);
    double (*Ys)[CBP] = reinterpret_cast<double (*)[CBP]>(csm + CB * CBP);
    const int p = blockIdx.x;
    const int nb = min(CB, K - j0);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const double* T = Tall + ((int64_t)p * ((K + CB - 1) / CB) + j0 / CB) * CB * CB;
    double* B = Ball + (int64_t)p * K * m + (int64_t)j0 * m;
    for (int e = tid; e < CB * CB; e += 256) {  // Xs[r][q] = T[q][r]
        const int q = e / CB, r = e % CB;
        Xs[r][q] = T[e];
    }
    double acc[4][4];
    for (int c0 = 0; c0 < m; c0 += CB) {
        const int nc = min(CB, m - c0);
        __syncthreads();
        for (int e = tid; e < CB * CB; e += 256) {  // Ys[col][q] = W[q][col]
            const int q = e / CB, c = e % CB;
            Ys[c][q] = (q < nb && c < nc) ? B[(int64_t)q * m + c0 + c] : 0.0;
        }
        __syncthreads();
        tile_update(Xs, Ys, nb, acc);
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2) {
            const int r = ty + 16 * a2;
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
                const int c = tx + 16 * b2;
                if (r < nb && c < nc) B[(int64_t)r * m + c0 + c] = acc[a2][b2];
            }
        }
    }
}

// back substitution update: W_i -= L_ji^T Z_j for row blocks i < j
// grid (i blocks * column chunks, P)
__global__ void __launch_bounds__(256)
k_back_update(int K, int m, int j0, const double* __restrict__ Aall, double* __restrict__ Ball) {
    extern __shared__ double csm[];
    double (*Xs)[CBP] = reinterpret_cast<double (*)[CBP]>(csm);  // Xs[r][q] = L[j0+q][i0+r]
    double (*Ys)[CBP] = reinterpret_cast<double (*)[CBP]>(csm + CB * CBP);  // Ys[c][q] = Z[j0+q][c0+c]
    const int p = blockIdx.y;
    const int nb = min(CB, K - j0);
    const int nmc = (m + CB - 1) / CB;
    const int bi = blockIdx.x / nmc, mc = blockIdx.x % nmc;
    const int i0 = bi * CB, c0 = mc * CB;
    if (i0 >= j0) return;
    const int ni = min(CB, j0 - i0);
    const double* A = Aall + (int64_t)p * K * K;
    double* B = Ball + (int64_t)p * K * m;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    for (int e = tid; e < CB * CB; e += 256) {
        const int q = e / CB, r = e % CB;  // coalesced over r (row j0+q of L)
        Xs[r][q] = (q < nb && r < ni) ? A[(int64_t)(j0 + q) * K + i0 + r] : 0.0;
        Ys[r][q] = (q < nb && c0 + r < m) ? B[(int64_t)(j0 + q) * m + c0 + r] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
    tile_update(Xs, Ys, nb, acc);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int gr = i0 + ty + 16 * a;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int gc = c0 + tx + 16 * b;
            if (gr < i0 + ni && gc < m) B[(int64_t)gr * m + gc] -= acc[a][b];
        }
    }
}

// out[p] = sum of squares of the (K*m) block of shard p (fixed order)
__global__ void __launch_bounds__(256) k_sumsq(int64_t n, const double* __restrict__ X, double* __restrict__ out) {
    __shared__ double sh[256];
    const double* x = X + (int64_t)blockIdx.x * n;
    double s = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += 256) s = fma(x[e], x[e], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

// =============================================================================
// Single-launch clustered solve for K <= 4*64 (the MOD shapes of the paper's
// split-and-merge runs). One thread-block cluster of NC = ceil(K/64) CTAs per
// shard; CTA c keeps block row c of A (tiles (c, 0..c), 64 x 64 FP64) in its
// shared memory for the whole solve, and the CTAs exchange panels through
// distributed shared memory (DSMEM). Instead of cluster-wide barriers every
// published object (T_J, L_cJ, W_J, Z_J) has a ready flag in its producer's
// shared memory, so each CTA runs ahead as far as its own inputs allow (the
// next CTA to factor defers its RHS update until after its factorisation):
//   forward, J = 0..NC-1:
//     CTA J    : factor A_JJ and form T_J = L_JJ^-1 in the same register sweep
//                (T overwrites the tile; L_JJ itself is never needed again),
//                W_J = T_J B_J
//     CTA c > J: L_cJ = A_cJ T_J^T (T_J read from CTA J)
//     CTA c > J: A_cK -= L_cJ L_KJ^T (J < K <= c, L_KJ from CTA K),
//                B_c -= L_cJ W_J
//   backward, J = NC-1..0:
//     CTA J    : Z_J = T_J^T W_J
//     CTA c < J: W_c -= L_Jc^T Z_J (L_Jc read from CTA J)
// Unused-atom masking, the pivot tolerance and ||W||^2 are folded in; every
// reduction runs in a fixed order (bitwise reproducible).
// =============================================================================
constexpr int CL_MAX = 4;
constexpr int TILE_D = CB * CBP;

// acc = X Y^T over q < nq on 64x64 smem tiles (rows padded to CBP);
// XT: X stored transposed (Xs[q][r])
template <bool XT>
__device__ __forceinline__ void tile_mm(const double* __restrict__ Xs, const double* __restrict__ Ys,
                                        int nq, double acc[4][4]) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int q = 0; q < nq; ++q) {
        double xv[4], yv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = XT ? Xs[q * CBP + ty + 16 * a] : Xs[(ty + 16 * a) * CBP + q];
#pragma unroll
        for (int b = 0; b < 4; ++b) yv[b] = Ys[(tx + 16 * b) * CBP + q];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(xv[a], yv[b], acc[a][b]);
    }
}

// S[col][q] = B[(row0 + q) * m + c0 + col] (q < nq, col < nc; zero padded)
__device__ __forceinline__ void stage_rows_t(double* __restrict__ S, const double* __restrict__ B, int m,
                                             int row0, int nq, int c0, int nc) {
    const int col = threadIdx.x & 63, qb = threadIdx.x >> 6;  // all 16 loads in flight
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int q = qb + 4 * k;
        v[k] = (q < nq && col < nc) ? B[(int64_t)(row0 + q) * m + c0 + col] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) S[col * CBP + qb + 4 * k] = v[k];
}

// 64 x CBP tile copy (e.g. from a peer CTA through DSMEM): every load of the
// thread is issued before the first store so the remote latency is paid once
__device__ __forceinline__ void copy_tile(double* __restrict__ dst, const double* src) {
    constexpr int N2 = TILE_D / 2, PER = (N2 + 255) / 256;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    double2 t[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int e = threadIdx.x + 256 * k;
        if (e < N2) t[k] = s2[e];
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int e = threadIdx.x + 256 * k;
        if (e < N2) d2[e] = t[k];
    }
}

// factor the 64x64 tile in place into T = L^-1, as a producer/consumer
// dataflow over columns (no CTA-wide barrier per column):
//   ownership: warp w owns columns q = w (mod 8), lane l rows l and l + 32
//              (16 entries of A/L and 16 of T per thread, in registers);
//   column k is produced by its owner warp as soon as its own entries have
//   received update k-1: the RAW column a_k (rows > k, zero elsewhere) and
//   the pivot d_k go to a ring slot in shared memory, signalled by an
//   mbarrier ("full"); no square root on this path: every warp forms
//   rd_k = 1/d_k itself (0 for a dependent pivot or a padding row), and
//   applies, for each owned entry (unconditional FMAs: the operands are zero
//   where the update must not act, or the entry is never read again),
//     the Cholesky rank-1 step   v_rq -= (a_r rd_k) a_q   (= l_r l_q), and
//     the inverse step           P_r  -= (a_r rd_k) P_k,
//   with P the unscaled rows of T (T_r = P_r / sqrt(d_r), applied at the
//   end); row k of P lives in the warp's lane k % 32 and is broadcast by
//   shuffles. A slot is released through an "empty" mbarrier (256 threads).
// The producer of column k+1 updates that column first and publishes before
// the rest of its work, so the critical path per column is one mbarrier
// hand-off, the reciprocal, one FMA and the store.
constexpr int FNB = 4;           // ring slots
constexpr int FSLOT = CB + 2;    // 64 raw values + d_k (+ pad)

__device__ __forceinline__ double inv_sqrt_f64(double d) {
    double y = (double)rsqrtf((float)fmax(d, 1e-300));
    y = y * fma(-0.5 * d * y, y, 1.5);
    return y * fma(-0.5 * d * y, y, 1.5);
}

__device__ __forceinline__ double rcp_f64(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    y = fma(y, fma(-d, y, 1.0), y);
    return fma(y, fma(-d, y, 1.0), y);
}

__device__ __forceinline__ void mbar_init_cta(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t* b, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

// ring: FNB x FSLOT doubles; bars: 2 * FNB mbarriers (full, empty); dval:
// CB doubles (pivots). The caller has synchronised the CTA after writing Ts.
__device__ __forceinline__ void factor_inverse(double* Ts, int nr, double tl, double* ring, uint64_t* bars,
                                               double* dval, int8_t* sdep) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint64_t* full = bars;
    uint64_t* empty = bars + FNB;
    if (tid == 0) {
        for (int b = 0; b < FNB; ++b) {
            mbar_init_cta(&full[b], 32);
            mbar_init_cta(&empty[b], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    double v[8][2], tv[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h, q = 8 * c + w;
            v[c][h] = (q <= r) ? Ts[r * CBP + q] : 0.0;
            tv[c][h] = (q == r) ? 1.0 : 0.0;
        }
    __syncthreads();  // barriers initialised
    // produce column k (called by warp k % 8 with its column entries final)
    auto produce = [&](int k, double x0, double x1) {  // x0, x1: this lane's entries of column k
        const int slot = k % FNB;
        if (k >= FNB) mbar_wait_cta(&empty[slot], ((k / FNB) - 1) & 1);
        double* col = ring + slot * FSLOT;
        col[lane] = (lane > k) ? x0 : 0.0;
        col[lane + 32] = (lane + 32 > k) ? x1 : 0.0;
        if (lane == (k & 31)) {
            const double d = (k < 32) ? x0 : x1;
            col[CB] = d;
            dval[k] = d;
        }
        mbar_arrive_cta(&full[slot]);
    };
    if (w == 0) produce(0, v[0][0], v[0][1]);
    // the two halves k < 32 / k >= 32 are separate loops so that k >> 5 is a
    // compile-time constant: for k >= 32 rows < 32 are finished (their a_r is
    // 0) and columns < 32 of L are dead; for k < 32 row k of P is zero in
    // columns >= 32. Those updates are skipped statically.
    auto step = [&](int kb, int kk, auto H) {
        constexpr int hk = decltype(H)::value;
        const int k = kb + kk;  // column k, owned by warp kk
        const int slot = k % FNB;
        mbar_wait_cta(&full[slot], (k / FNB) & 1);
        const double* col = ring + slot * FSLOT;
        const double d = col[CB];
        const double rd = (!(d > tl) || k >= nr) ? 0.0 : rcp_f64(d);
        const double lr0 = hk == 0 ? col[lane] * rd : 0.0;
        const double lr1 = col[lane + 32] * rd;
        double lq[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) lq[c] = (hk == 0 || c >= 4) ? col[8 * c + w] : 0.0;
        const int nk = k + 1, nw = (kk + 1) & 7, nc = nk >> 3;
        if (nk < CB && w == nw) {
            double x0 = 0.0, x1 = 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c == nc) {
                    if (hk == 0) v[c][0] = fma(-lr0, lq[c], v[c][0]);
                    v[c][1] = fma(-lr1, lq[c], v[c][1]);
                    lq[c] = 0.0;  // applied
                    x0 = v[c][0];
                    x1 = v[c][1];
                }
            produce(nk, x0, x1);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (hk == 1 && c < 4) continue;  // dead columns of L
            if (hk == 0) v[c][0] = fma(-lr0, lq[c], v[c][0]);
            v[c][1] = fma(-lr1, lq[c], v[c][1]);
        }
        // row k of P (final: every earlier row has been applied to it)
        const int lk = k & 31;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (hk == 0 && c >= 4) continue;  // zero right of the diagonal
            const double tk = __shfl_sync(SDB_FULL, tv[c][hk], lk);
            if (hk == 0) tv[c][0] = fma(-lr0, tk, tv[c][0]);
            tv[c][1] = fma(-lr1, tk, tv[c][1]);
        }
        mbar_arrive_cta(&empty[slot]);
    };
#pragma unroll 1
    for (int kb = 0; kb < 32; kb += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) step(kb, kk, std::integral_constant<int, 0>{});
    }
#pragma unroll 1
    for (int kb = 32; kb < CB; kb += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) step(kb, kk, std::integral_constant<int, 1>{});
    }
    __syncthreads();
    // T_r = P_r / sqrt(d_r) (0 for dependent pivots / padding rows)
    if (tid < CB) {
        const double d = dval[tid];
        const bool dep = !(d > tl) || tid >= nr;
        sdep[tid] = dep ? 1 : 0;
        dval[tid] = dep ? 0.0 : inv_sqrt_f64(d);
    }
    __syncthreads();
    const double s0 = dval[lane], s1 = dval[lane + 32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        Ts[lane * CBP + 8 * c + w] = tv[c][0] * s0;
        Ts[(lane + 32) * CBP + 8 * c + w] = tv[c][1] * s1;
    }
}

// fixed-order CTA sum / max of one double per thread
__device__ __forceinline__ double block_reduce(double x, double* red, bool is_max) {
    red[threadIdx.x] = x;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            red[threadIdx.x] = is_max ? fmax(red[threadIdx.x], red[threadIdx.x + w])
                                      : red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// ready flags live in the producer's shared memory: written once per launch
// with release semantics at cluster scope (after a CTA barrier, so the whole
// CTA's smem / global writes are covered); consumers poll them with acquire
// loads through the DSMEM window, then barrier.
__device__ __forceinline__ void flag_publish(int* f) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
}
__device__ __forceinline__ void flag_wait(const int* remote) {
    if (threadIdx.x == 0) {
        unsigned v = 0;
        do {
            asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(v) : "l"(remote) : "memory");
        } while (v == 0);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256, 1)
k_chol_cluster(int K, int m, double* __restrict__ Aall, double* __restrict__ Ball,
               const int32_t* __restrict__ usage, double rel_tol, int8_t* __restrict__ depmask,
               int32_t* __restrict__ ndep, double* __restrict__ wsq) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double xsm[];
    __shared__ __align__(16) double fring[FNB * FSLOT];
    __shared__ uint64_t fbars[2 * FNB];
    __shared__ double fdval[CB];
    __shared__ double red[256];
    __shared__ double s_part[2];  // [0] diag max, [1] ||W||^2 of this block row
    __shared__ int8_t s_use[CL_MAX * CB];
    __shared__ int8_t sdep[CB];
    __shared__ int s_nd;
    // fT: T_c ready; fW: W_c ready; fZ: Z_c ready; fL[J]: L_cJ ready
    __shared__ int fT, fW, fZ, fL[CL_MAX];
    const int NC = (int)cl.num_blocks();
    const int c = (int)cl.block_rank();
    const int p = blockIdx.x / NC;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int r0 = c * CB, nr = min(CB, K - r0);
    const double* A = Aall + (int64_t)p * K * K;
    double* B = Ball + (int64_t)p * K * m;
    const int32_t* use = usage + (int64_t)p * K;
    double* S1 = xsm + NC * TILE_D;
    double* S2 = S1 + TILE_D;
    auto tile = [&](int J) { return xsm + J * TILE_D; };
    auto nrows = [&](int J) { return min(CB, K - J * CB); };
    double acc[4][4];

    if (tid == 0) {
        fT = fW = fZ = 0;
        for (int J = 0; J < CL_MAX; ++J) fL[J] = 0;
    }
    // ---- load block row c with unused atoms masked to the identity
    for (int q = tid; q < NC * CB; q += 256) s_use[q] = (q < K && use[q]) ? 1 : 0;
    __syncthreads();
    {
        const int q = tid & 63, rb = tid >> 6;  // column q of every tile, rows rb + 4k
        for (int J = 0; J <= c; ++J) {
            double* T = tile(J);
            const int gq = J * CB + q;
            double v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int gr = r0 + rb + 4 * k;
                const bool ld = s_use[gq] && gr < K && s_use[gr];
                v[k] = ld ? A[(int64_t)gr * K + gq] : ((gr == gq) ? 1.0 : 0.0);
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) T[(rb + 4 * k) * CBP + q] = v[k];
        }
    }
    {
        double mx = 0.0;
        if (tid < nr && use[r0 + tid]) mx = A[(int64_t)(r0 + tid) * K + r0 + tid];
        mx = block_reduce(mx, red, true);
        if (tid == 0) { s_part[0] = mx; s_part[1] = 0.0; s_nd = 0; }
    }
    cl.sync();  // flags initialised and diagonal maxima published everywhere
    double dmax = 0.0;
    for (int k = 0; k < NC; ++k) dmax = fmax(dmax, cl.map_shared_rank(s_part, k)[0]);
    const double tl = rel_tol * dmax;

    // B_c -= L_cJ W_J (W_J rows of block J, published by CTA J)
    auto b_update = [&](int J) {
        flag_wait(cl.map_shared_rank(&fW, J));
        const int nJ = nrows(J);
        for (int c0 = 0; c0 < m; c0 += CB) {
            const int nc = min(CB, m - c0);
            __syncthreads();
            stage_rows_t(S1, B, m, J * CB, nJ, c0, nc);
            __syncthreads();
            tile_mm<false>(tile(J), S1, nJ, acc);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int rr = ty + 16 * a, cc = tx + 16 * b;
                    if (rr < nr && cc < nc) B[(int64_t)(r0 + rr) * m + c0 + cc] -= acc[a][b];
                }
        }
    };

    // ---- forward: panels of the block columns left of the diagonal
    bool b_pending[CL_MAX] = {false, false, false, false};
    for (int J = 0; J < c; ++J) {
        const int nJ = nrows(J);
        flag_wait(cl.map_shared_rank(&fT, J));
        copy_tile(S1, cl.map_shared_rank(tile(J), J));
        __syncthreads();
        tile_mm<false>(tile(J), S1, nJ, acc);  // L_cJ = A_cJ T_J^T
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) tile(J)[(ty + 16 * a) * CBP + tx + 16 * b] = acc[a][b];
        flag_publish(&fL[J]);
        // trailing tiles of this block row, next panel column first
        for (int Kb = J + 1; Kb <= c; ++Kb) {
            const double* Ly = tile(J);
            if (Kb != c) {
                flag_wait(cl.map_shared_rank(&fL[J], Kb));
                copy_tile(S1, cl.map_shared_rank(tile(J), Kb));
                Ly = S1;
            }
            __syncthreads();
            tile_mm<false>(tile(J), Ly, nJ, acc);
            double* T = tile(Kb);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) T[(ty + 16 * a) * CBP + tx + 16 * b] -= acc[a][b];
            __syncthreads();
        }
        // the next CTA to factor keeps the RHS update off its critical path
        if (c > J + 1) b_update(J);
        else b_pending[J] = true;
    }
    // ---- own diagonal block: T_c = L_cc^-1
    factor_inverse(tile(c), nr, tl, fring, fbars, fdval, sdep);
    if (tid < nr) depmask[(int64_t)p * K + r0 + tid] = sdep[tid];
    if (tid == 0) {
        int nd = 0;
        for (int q = 0; q < nr; ++q) nd += sdep[q];
        s_nd = nd;
    }
    flag_publish(&fT);
    double wloc = 0.0;
    if (m <= CB) {
        // one column chunk: the deferred RHS update (B_c -= L_cJ W_J, on this
        // CTA's critical path) is applied in registers and W_c = T_c B_c
        // formed from them, without a global round trip
        double br[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                br[a][b] = (rr < nr && cc < m) ? B[(int64_t)(r0 + rr) * m + cc] : 0.0;
            }
        for (int J = 0; J < c; ++J) {
            if (!b_pending[J]) continue;
            flag_wait(cl.map_shared_rank(&fW, J));
            stage_rows_t(S1, B, m, J * CB, nrows(J), 0, m);
            __syncthreads();
            tile_mm<false>(tile(J), S1, nrows(J), acc);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) br[a][b] -= acc[a][b];
            __syncthreads();
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) S1[(tx + 16 * b) * CBP + ty + 16 * a] = br[a][b];
        __syncthreads();
        tile_mm<false>(tile(c), S1, nr, acc);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                if (rr < nr && cc < m) {
                    B[(int64_t)(r0 + rr) * m + cc] = acc[a][b];
                    wloc = fma(acc[a][b], acc[a][b], wloc);
                }
            }
    } else {
    for (int J = 0; J < c; ++J)
        if (b_pending[J]) b_update(J);
    // W_c = T_c B_c
    for (int c0 = 0; c0 < m; c0 += CB) {
        const int nc = min(CB, m - c0);
        __syncthreads();
        stage_rows_t(S1, B, m, r0, nr, c0, nc);
        __syncthreads();
        tile_mm<false>(tile(c), S1, nr, acc);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                if (rr < nr && cc < nc) {
                    B[(int64_t)(r0 + rr) * m + c0 + cc] = acc[a][b];
                    wloc = fma(acc[a][b], acc[a][b], wloc);
                }
            }
    }
    }
    flag_publish(&fW);
    wloc = block_reduce(wloc, red, false);
    if (tid == 0) s_part[1] = wloc;

    // ---- backward: W_c -= L_Jc^T Z_J for J > c, then Z_c = T_c^T W_c
    if (m <= CB) {
        // one column chunk: W_c stays in registers across the J updates (no
        // global read-modify-write per link, no restaging for Z_c), and L_Jc
        // is copied before Z_J is waited for
        double wr[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                wr[a][b] = (rr < nr && cc < m) ? B[(int64_t)(r0 + rr) * m + cc] : 0.0;
            }
        for (int J = NC - 1; J > c; --J) {
            const int nJ = nrows(J);
            flag_wait(cl.map_shared_rank(&fL[c], J));
            copy_tile(S2, cl.map_shared_rank(tile(c), J));  // L_Jc (rows of block J)
            flag_wait(cl.map_shared_rank(&fZ, J));
            stage_rows_t(S1, B, m, J * CB, nJ, 0, m);
            __syncthreads();
            tile_mm<true>(S2, S1, nJ, acc);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) wr[a][b] -= acc[a][b];
            __syncthreads();
        }
        // S1[col][q] = W_c[q][col] (the stage_rows_t layout)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) S1[(tx + 16 * b) * CBP + ty + 16 * a] = wr[a][b];
        __syncthreads();
        tile_mm<true>(tile(c), S1, nr, acc);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                if (rr < nr && cc < m) B[(int64_t)(r0 + rr) * m + cc] = acc[a][b];
            }
        flag_publish(&fZ);
        cl.sync();
        if (c == 0 && tid == 0) {
            double w = 0.0;
            int nd = 0;
            for (int k = 0; k < NC; ++k) {
                w += cl.map_shared_rank(s_part, k)[1];
                nd += *cl.map_shared_rank(&s_nd, k);
            }
            if (wsq) wsq[p] = w;
            ndep[p] = nd;
        }
        cl.sync();  // keep every CTA's shared memory alive until rank 0 has read it
        return;
    }
    for (int J = NC - 1; J > c; --J) {
        const int nJ = nrows(J);
        flag_wait(cl.map_shared_rank(&fZ, J));
        copy_tile(S2, cl.map_shared_rank(tile(c), J));  // L_Jc (rows of block J)
        for (int c0 = 0; c0 < m; c0 += CB) {
            const int nc = min(CB, m - c0);
            __syncthreads();
            stage_rows_t(S1, B, m, J * CB, nJ, c0, nc);
            __syncthreads();
            tile_mm<true>(S2, S1, nJ, acc);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int rr = ty + 16 * a, cc = tx + 16 * b;
                    if (rr < nr && cc < nc) B[(int64_t)(r0 + rr) * m + c0 + cc] -= acc[a][b];
                }
        }
    }
    for (int c0 = 0; c0 < m; c0 += CB) {
        const int nc = min(CB, m - c0);
        __syncthreads();
        stage_rows_t(S1, B, m, r0, nr, c0, nc);
        __syncthreads();
        tile_mm<true>(tile(c), S1, nr, acc);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int rr = ty + 16 * a, cc = tx + 16 * b;
                if (rr < nr && cc < nc) B[(int64_t)(r0 + rr) * m + c0 + cc] = acc[a][b];
            }
    }
    flag_publish(&fZ);
    cl.sync();
    if (c == 0 && tid == 0) {
        double w = 0.0;
        int nd = 0;
        for (int k = 0; k < NC; ++k) {
            w += cl.map_shared_rank(s_part, k)[1];
            nd += *cl.map_shared_rank(&s_nd, k);
        }
        if (wsq) wsq[p] = w;
        ndep[p] = nd;
    }
    cl.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

static int chol_solve_cluster(int P, int K, int m, double* A, double* B, const int32_t* usage,
                              double rel_tol, int8_t* depmask, int32_t* ndep, double* wsq, cudaStream_t st) {
    const int NC = (K + CB - 1) / CB;
    const int smem = (NC + 2) * TILE_D * (int)sizeof(double);
    {
        cudaError_t e = set_max_smem((const void*)k_chol_cluster, smem);
        if (e != cudaSuccess) return (int)e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P * NC));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)NC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k_chol_cluster, K, m, A, B, usage, rel_tol, depmask, ndep, wsq);
}

int64_t chol_ws_bytes(int P, int K) {
    const int64_t nblk = (K + CB - 1) / CB;
    return (int64_t)P * nblk * CB * CB * sizeof(double) + (int64_t)P * sizeof(double) + 512;
}

int chol_solve(int P, int K, int m, double* A, double* B, const int32_t* usage, double rel_tol,
               int8_t* depmask, int32_t* ndep, double* wsq, void* ws, cudaStream_t st) {
    static const bool force_chain = getenv("SDB_CHOL_CHAIN") != nullptr;  // A/B switch for tests
    if (K <= CL_MAX * CB && P > 0 && !force_chain)
        return chol_solve_cluster(P, K, m, A, B, usage, rel_tol, depmask, ndep, wsq, st);
    const int64_t nblk = (K + CB - 1) / CB;
    double* T = (double*)ws;
    double* tol = T + (int64_t)P * nblk * CB * CB;
    const int smem2 = 2 * CB * CBD * (int)sizeof(double);
    const int smemP = 2 * CB * CBP * (int)sizeof(double);
    const int smemD = (2 * CB * CBP + 32 * 33) * (int)sizeof(double);
    {
        cudaError_t e = set_max_smem((const void*)k_chol_update, smem2);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_back_update, smem2);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_chol_panel, smemP);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_back_diag, smemP);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_chol_diag, smemD);
        if (e != cudaSuccess) return (int)e;
    }
    {
        const int64_t KK = (int64_t)K * K;
        dim3 g((unsigned)std::min<int64_t>(64, (KK + 255) / 256), (unsigned)P);
        k_chol_prep<<<g, 256, 0, st>>>(K, A, usage, rel_tol, tol, ndep);
    }
    const int nmc = (m + CB - 1) / CB;
    for (int j0 = 0; j0 < K; j0 += CB) {
        const int nb = std::min(CB, K - j0);
        k_chol_diag<<<P, 256, smemD, st>>>(K, j0, A, T, tol, depmask, ndep);
        const int rows_below = K - j0 - nb;
        dim3 gp((unsigned)(1 + (rows_below + CB - 1) / CB), (unsigned)P);
        k_chol_panel<<<gp, 256, smemP, st>>>(K, m, j0, A, B, T);
        const int nt = (rows_below + CB - 1) / CB;
        const int tiles = nt * (nt + 1) / 2 + nt * nmc;
        if (tiles > 0) {
            dim3 gu((unsigned)tiles, (unsigned)P);
            k_chol_update<<<gu, 256, smem2, st>>>(K, m, j0, A, B);
        }
    }
    if (wsq) k_sumsq<<<P, 256, 0, st>>>((int64_t)K * m, B, wsq);
    const int last = (int)((nblk - 1) * CB);
    for (int j0 = last; j0 >= 0; j0 -= CB) {
        k_back_diag<<<P, 256, smemP, st>>>(K, m, j0, T, B);
        if (j0 > 0) {
            const int ib = (j0 + CB - 1) / CB;
            dim3 gb((unsigned)(ib * nmc), (unsigned)P);
            k_back_update<<<gb, 256, smem2, st>>>(K, m, j0, A, B);
        }
    }
    return (int)cudaGetLastError();
}

}  // namespace sdb
