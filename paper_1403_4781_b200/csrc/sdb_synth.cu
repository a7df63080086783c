// On-device synthetic sparse-model signals (the generator the
// reference runs on the host, synthesis.py:56-79 gen_signals, plus the
// additive noise BASELINE.json's configs add).
//
// Signal i: s distinct atoms drawn uniformly from K, standard-normal
// coefficients, y = sum_t c_t d_{a_t} + sigma * n with n ~ N(0, I_m).
// Randomness is counter-based (Philox4x32-10 keyed by the seed, counter =
// (signal, draw index)), so every signal is a fixed function of (seed, i):
// the result does not depend on the launch shape, and the CPU oracle is fed
// the very same array (copied back), which replaces bit-compatibility with
// the host's PCG64 stream. Normals by Box-Muller in FP64; sums in FP64,
// stored in the working precision.
//
// Layout: one warp per signal; lane 0 draws the support (rejection of
// repeats, deterministic order) and the coefficients, the warp forms the
// m-vector (lane owns components lane, lane+32, ...) from the f64 atom-major
// dictionary. HBM-bound on the output (4m or 8m bytes per signal).
#include <algorithm>
#include <cstdint>

#include "sdb_common.cuh"
#include "sdb_internal.h"

namespace sdb {
namespace {

struct Philox {
    uint32_t k0, k1;
    __device__ __forceinline__ uint4 operator()(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) const {
        uint32_t a = k0, b = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
            const uint32_t n0 = hi1 ^ c1 ^ a, n1 = lo1, n2 = hi0 ^ c3 ^ b, n3 = lo0;
            c0 = n0; c1 = n1; c2 = n2; c3 = n3;
            a += 0x9E3779B9u;
            b += 0xBB67AE85u;
        }
        return make_uint4(c0, c1, c2, c3);
    }
};

// two standard normals from one Philox block (draw index j of signal i, stream tag)
__device__ __forceinline__ double2 normals(const Philox& ph, int64_t i, uint32_t j, uint32_t tag) {
    const uint4 r = ph((uint32_t)i, (uint32_t)(i >> 32), j, tag);
    const uint64_t bits = (((uint64_t)r.x << 32) | r.y) >> 11;           // 53 random bits
    const double u1 = ((double)bits + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
    const double u2 = (double)r.z * (1.0 / 4294967296.0);                 // [0, 1)
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    return make_double2(rad * cs, rad * sn);
}

constexpr int SY_MAX_S = 64;

template <typename T>
__global__ void __launch_bounds__(256)
k_synth_sparse(int64_t N, int m, int K, int s, const double* __restrict__ D, double sigma, Philox ph,
               T* __restrict__ Y, int64_t ldy, int32_t* __restrict__ sup_out) {
    __shared__ int s_sup[8][SY_MAX_S];
    __shared__ double s_coef[8][SY_MAX_S];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t i = (int64_t)blockIdx.x * 8 + wib; i < N; i += nwarps) {
        if (lane == 0) {
            // s distinct atoms: uniform draws (32-bit multiply-shift), repeats
            // rejected (fixed order)
            uint32_t j = 0;
            int n = 0;
            while (n < s) {
                const uint4 r = ph((uint32_t)i, (uint32_t)(i >> 32), j++, 0x5u);
                const uint32_t v[4] = {r.x, r.y, r.z, r.w};
                for (int q = 0; q < 4 && n < s; ++q) {
                    const int a = (int)(((uint64_t)v[q] * (uint64_t)K) >> 32);
                    bool dup = false;
                    for (int t = 0; t < n; ++t) dup |= s_sup[wib][t] == a;
                    if (!dup) s_sup[wib][n++] = a;
                }
            }
            for (int t = 0; t < s; t += 2) {
                const double2 z = normals(ph, i, (uint32_t)t, 0x6u);
                s_coef[wib][t] = z.x;
                if (t + 1 < s) s_coef[wib][t + 1] = z.y;
            }
        }
        __syncwarp();
        for (int c0 = 0; c0 < m; c0 += 64) {
            // noise for components c0 + 2*lane, c0 + 2*lane + 1
            const double2 z = normals(ph, i, (uint32_t)(c0 / 64 * 32 + lane), 0x7u);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = c0 + 2 * lane + h;
                if (c < m) {
                    double acc = 0.0;
                    for (int t = 0; t < s; ++t) acc = fma(s_coef[wib][t], D[(int64_t)s_sup[wib][t] * m + c], acc);
                    acc = fma(sigma, h ? z.y : z.x, acc);
                    Y[i * ldy + c] = (T)acc;
                }
            }
        }
        if (sup_out != nullptr)
            for (int t = lane; t < s; t += 32) sup_out[i * s + t] = s_sup[wib][t];
        __syncwarp();
    }
}

}  // namespace

int synth_sparse(int dtype_f64, int64_t N, int m, int K, int s, const double* D, double sigma, uint64_t seed,
                 void* Y, int64_t ldy, int32_t* sup_out, cudaStream_t st) {
    if (s < 1 || s > SY_MAX_S || s > K || m < 1 || ldy < m) return (int)cudaErrorInvalidValue;
    if (N <= 0) return 0;
    Philox ph{(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int64_t blocks = std::min<int64_t>((N + 7) / 8, 148 * 64);
    if (dtype_f64)
        k_synth_sparse<double><<<(unsigned)blocks, 256, 0, st>>>(N, m, K, s, D, sigma, ph, (double*)Y, ldy, sup_out);
    else
        k_synth_sparse<float><<<(unsigned)blocks, 256, 0, st>>>(N, m, K, s, D, sigma, ph, (float*)Y, ldy, sup_out);
    return (int)cudaGetLastError();
}

}  // namespace sdb
