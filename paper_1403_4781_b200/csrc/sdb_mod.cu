// MOD dictionary update, degenerate-atom replacement and residual norms on
// B200, batched over P shards (one launch per phase covers every shard).
//
// Reference: /root/reference/pkg/src/sparsedict/dictionary_update.py
//   mod_update :72-114, replace_degenerate_atoms :117-177, normalize :56-69
// and metrics.py:30-44 (mse_db), trainer.py:138-162,248-256 (init / merge).
//
// Determinism: no floating-point atomics anywhere. The codes are
// counting-sorted into per-(shard, atom) buckets with a fixed order (integer
// atomics only for counts), then every normal-equation entry is a sequential
// FP64 sum over its bucket. Results are bitwise reproducible run to run.
//
// Normal equations per shard:  A = X X^T (K x K), B = (Y X^T)^T (K x m)
// solved as A Z = B with an FP64 blocked Cholesky (unused atoms masked to the
// identity, which equals the minimum-norm lstsq solution on the used block);
// D_new = Z^T (atom-major storage == Z row-major).
#include <cfloat>
#include <type_traits>

#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_mod.h"
#include "sdb_chol.h"

namespace sdb {

// signals per chunk (chunks never straddle shards): aims at ~32 chunks per SM
// (256 signals for the C2 locals, down to one 32-signal warp group for the
// merge phase), so the per-chunk histogram / placement kernels always have
// enough parallel work; up to 1024 for very large jobs
__host__ __device__ inline int chunk_size(int64_t N) {
    int ch = 1024;
    while (ch > 32 && (int64_t)ch * 148 * 32 > N) ch >>= 1;
    return ch;
}

// chunk_first[p] = first chunk of shard p; chunk_first[P] = total chunks
__global__ void k_chunk_layout(const int64_t* __restrict__ off, int P, int CH, int64_t* __restrict__ cf) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t c = 0;
        for (int p = 0; p < P; ++p) {
            cf[p] = c;
            c += (off[p + 1] - off[p] + CH - 1) / CH;
        }
        cf[P] = c;
    }
}

struct ChunkInfo {
    int p;
    int64_t lo, hi;
};

__device__ __forceinline__ ChunkInfo chunk_info(const int64_t* off, const int64_t* cf, int P, int64_t c, int CH) {
    int lo = 0, hi = P - 1;
    while (lo < hi) {  // last p with cf[p] <= c (empty shards share cf values)
        int mid = (lo + hi + 1) >> 1;
        if (cf[mid] <= c) lo = mid; else hi = mid - 1;
    }
    ChunkInfo ci;
    ci.p = lo;
    ci.lo = off[lo] + (c - cf[lo]) * CH;
    ci.hi = min(ci.lo + CH, off[lo + 1]);
    return ci;
}

// ---- (a) per-chunk atom histograms: CTA per chunk, each thread a strided
// share of the chunk's signals, shared-memory integer atomics (counts are
// order-free)
__global__ void __launch_bounds__(256)
k_chunk_hist(const int64_t* __restrict__ off, const int64_t* __restrict__ cf, int P, int K, int cap, int CH,
             const int32_t* __restrict__ idx, const int32_t* __restrict__ counts,
             int32_t* __restrict__ chunk_hist) {
    extern __shared__ int32_t cnt[];
    const int64_t c = blockIdx.x;
    if (c >= cf[P]) return;
    for (int a = threadIdx.x; a < K; a += blockDim.x) cnt[a] = 0;
    __syncthreads();
    const ChunkInfo ci = chunk_info(off, cf, P, c, CH);
    for (int64_t i = ci.lo + threadIdx.x; i < ci.hi; i += blockDim.x) {
        const int n = counts[i];
        for (int t = 0; t < n; ++t) atomicAdd(&cnt[idx[i * cap + t]], 1);
    }
    __syncthreads();
    for (int a = threadIdx.x; a < K; a += blockDim.x) chunk_hist[c * K + a] = cnt[a];
}

// ---- (b) usage[p][a] = sum over the shard's chunks. Block = (shard, 32
// atoms); warp w sums the w-th eighth of the shard's chunks (lane = atom) and
// keeps that partial for (d).
constexpr int SCW = 16;  // warps splitting a shard's chunk range in the usage / offset scans

__device__ __forceinline__ void chunk_piece(const int64_t* cf, int p, int w, int64_t& c0, int64_t& c1) {
    const int64_t lo = cf[p], n = cf[p + 1] - lo;
    c0 = lo + n * w / SCW;
    c1 = lo + n * (w + 1) / SCW;
}

__global__ void __launch_bounds__(SCW * 32)
k_usage_from_chunks(const int64_t* __restrict__ cf, int P, int K, const int32_t* __restrict__ chunk_hist,
                    int64_t* __restrict__ wpart, int32_t* __restrict__ usage) {
    __shared__ int64_t part[SCW][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int p = blockIdx.y, a = blockIdx.x * 32 + lane;
    int64_t c0, c1;
    chunk_piece(cf, p, wib, c0, c1);
    int64_t s = 0;
    if (a < K)
        for (int64_t c = c0; c < c1; ++c) s += chunk_hist[c * K + a];
    part[wib][lane] = s;
    if (a < K) wpart[((int64_t)p * SCW + wib) * K + a] = s;
    __syncthreads();
    if (wib == 0 && a < K) {
        int64_t t = 0;
#pragma unroll
        for (int w = 0; w < SCW; ++w) t += part[w][lane];
        usage[(int64_t)p * K + a] = (int32_t)t;
    }
}

// ---- (d) chunk_off[c][a] = bucket_off[p][a] + prefix over earlier chunks
__global__ void __launch_bounds__(SCW * 32)
k_chunk_offsets(const int64_t* __restrict__ cf, int P, int K, const int32_t* __restrict__ chunk_hist,
                const int64_t* __restrict__ wpart, const int64_t* __restrict__ bucket_off,
                int64_t* __restrict__ chunk_off) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int p = blockIdx.y, a = blockIdx.x * 32 + lane;
    if (a >= K) return;
    int64_t run = bucket_off[(int64_t)p * K + a];
    for (int w = 0; w < wib; ++w) run += wpart[((int64_t)p * SCW + w) * K + a];
    int64_t c0, c1;
    chunk_piece(cf, p, wib, c0, c1);
    for (int64_t c = c0; c < c1; ++c) {
        chunk_off[c * K + a] = run;
        run += chunk_hist[c * K + a];
    }
}

__device__ __forceinline__ void load_row8(const int32_t* __restrict__ p, int (&v)[8]);

// ---- (e) stable placement: order inside a bucket = (chunk, 32-signal group,
// slot, lane) — a fixed function of the input.
template <typename T>
__global__ void __launch_bounds__(256)
k_place(const int64_t* __restrict__ off, const int64_t* __restrict__ cf, int P, int K, int cap, int CH,
        const int32_t* __restrict__ idx, const T* __restrict__ val, const int32_t* __restrict__ counts,
        const int64_t* __restrict__ chunk_off, int32_t* __restrict__ bent) {
    extern __shared__ int64_t sh_pos[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * 8 + wib;
    if (c >= cf[P]) return;
    int64_t* pos = sh_pos + (int64_t)wib * K;
    for (int a = lane; a < K; a += 32) pos[a] = chunk_off[c * K + a];
    __syncwarp();
    const ChunkInfo ci = chunk_info(off, cf, P, c, CH);
    // one (slot t) round of a 32-signal group: lanes with the same atom take
    // consecutive positions in lane order
    auto round = [&](int64_t i, int t, bool act, int a) {
        const unsigned am = __ballot_sync(SDB_FULL, act);
        unsigned peers = 0;
        int64_t base = 0;
        if (act) {
            peers = __match_any_sync(am, a);
            base = pos[a];
        }
        __syncwarp();
        if (act) {
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int64_t q = base + rank;
            bent[q] = (int32_t)(i * cap + t);  // flat code index: signal i, slot t
            if (rank == 0) pos[a] = base + __popc(peers);
        }
        __syncwarp();
    };
    const bool row8 = cap == 8 && (reinterpret_cast<uintptr_t>(idx) & 15) == 0;
    if (row8) {
        // the whole index row of every signal of the group (and of the next
        // group) is requested before its eight rounds, instead of one
        // dependent load in front of every round
        int nn = 0, an[8];
        auto fetch = [&](int64_t i, int& n, int (&as)[8]) {
            n = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) as[t] = 0;
            if (i < ci.hi) {
                n = counts[i];
                load_row8(idx + i * 8, as);
            }
        };
        fetch(ci.lo + lane, nn, an);
        for (int64_t g = ci.lo; g < ci.hi; g += 32) {
            const int64_t i = g + lane;
            const int n = nn;
            int as[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) as[t] = an[t];
            fetch(i + 32, nn, an);
            const int nmax = __reduce_max_sync(SDB_FULL, n);
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (t < nmax) round(i, t, t < n, as[t]);   // warp-uniform
        }
        return;
    }
    for (int64_t g = ci.lo; g < ci.hi; g += 32) {
        const int64_t i = g + lane;
        const int n = (i < ci.hi) ? counts[i] : 0;
        const int nmax = __reduce_max_sync(SDB_FULL, n);
        for (int t = 0; t < nmax; ++t) {
            const bool act = t < n;
            round(i, t, act, act ? idx[i * cap + t] : 0);
        }
    }
}

// ---- (f+g) both normal-equation rows of one bucket in one pass. CTA per
// (shard p, atom a), 8 warps; warp w takes the bucket's 32-entry batches
// w, w+8, ... and per batch
//   B[p][a][:] += sum y_i x_ai   (four signal rows in flight, as k_yxt),
//   A[p][a][:] += sum x_ai x_i   (diagonal as one warp sum; the other atoms
//                                 of multi-atom code rows in lane-parallel
//                                 rounds, collisions in lane order, as k_xxt)
// so the X X^T work hides under the Y-row gathers and the bucket is read
// once. Per-warp partials are combined in warp order: the result is a fixed
// function of the input (bitwise that of the separate kernels).
template <typename TY, typename T, int MPL>
__global__ void __launch_bounds__(256)
k_normal_eq(int P, int K, int m, const TY* __restrict__ Y, int64_t ldy, const int64_t* __restrict__ bucket_off,
            int cap, const int32_t* __restrict__ idx, const T* __restrict__ val,
            const int32_t* __restrict__ counts, const int32_t* __restrict__ bent, double* __restrict__ B,
            double* __restrict__ A) {
    extern __shared__ double sh_row[];  // 8 warps x K (X X^T row partials), then 8 x 32*MPL (Y X^T)
    double (*part)[MPL * 32] = reinterpret_cast<double (*)[MPL * 32]>(sh_row + 8 * (int64_t)K);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const bool y2 = MPL == 2 && std::is_same<TY, float>::value && m == 64 && (ldy & 1) == 0 &&
                    (reinterpret_cast<uintptr_t>(Y) & 7) == 0;
    const int64_t e = blockIdx.x;  // (p, a)
    const int self = (int)(e % K);
    double* row = sh_row + (int64_t)wib * K;
    for (int b = lane; b < K; b += 32) row[b] = 0.0;
    __syncwarp();
    double acc[MPL];
#pragma unroll
    for (int q = 0; q < MPL; ++q) acc[q] = 0.0;
    double diag = 0.0;
    const int64_t lo = bucket_off[e], hi = bucket_off[e + 1];
    for (int64_t b0 = lo + 32 * wib; b0 < hi; b0 += 32 * 8) {
        const int nbat = (int)min((int64_t)32, hi - b0);
        const int my_e = lane < nbat ? bent[b0 + lane] : 0;
        const int my_sig = my_e / cap;
        const double my_val = lane < nbat ? (double)val[my_e] : 0.0;
        const int my_n = lane < nbat ? counts[my_sig] : 0;
        // Y X^T (64-value float rows: lane l walks columns 2l, 2l + 1 with one
        // 8-byte load per entry)
        if (y2) {
            if constexpr (MPL == 2 && std::is_same<TY, float>::value) {
                for (int j = 0; j < nbat; j += 4) {
                    float2 yv[4];
                    const bool full = j + 4 <= nbat;   // warp-uniform
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = __shfl_sync(SDB_FULL, my_sig, (j + u) & 31);
                        yv[u] = make_float2(0.f, 0.f);
                        if (full || j + u < nbat)
                            yv[u] = __ldg(reinterpret_cast<const float2*>(Y + (int64_t)i * ldy) + lane);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double v = __shfl_sync(SDB_FULL, my_val, (j + u) & 31);
                        acc[0] = fma((double)yv[u].x, v, acc[0]);
                        acc[1] = fma((double)yv[u].y, v, acc[1]);
                    }
                }
            }
        } else
        for (int j = 0; j < nbat; j += 4) {
            double yv[4][MPL];
            double vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = __shfl_sync(SDB_FULL, my_sig, (j + u) & 31);
                vv[u] = __shfl_sync(SDB_FULL, my_val, (j + u) & 31);
                const TY* y = Y + (int64_t)i * ldy;
#pragma unroll
                for (int q = 0; q < MPL; ++q) {
                    const int r = lane + 32 * q;
                    yv[u][q] = (j + u < nbat && r < m) ? (double)y[r] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < MPL; ++q) acc[q] = fma(yv[u][q], vv[u], acc[q]);
        }
        // X X^T: a single-atom code row holds only this bucket's atom, whose
        // contribution is the diagonal term
        diag += warp_sum(my_val * my_val);
        const int my_no = my_n > 1 ? my_n : 0;
        const int nmax = (int)__reduce_max_sync(SDB_FULL, (unsigned)my_no);
        // slot t + 1's index and value are requested before slot t's rounds
        int bn = -1;
        double cn = 0.0;
        if (0 < my_no) {
            bn = idx[(int64_t)my_sig * cap];
            cn = (double)val[(int64_t)my_sig * cap];
        }
        for (int t = 0; t < nmax; ++t) {
            int b = -1;
            double c = 0.0;
            if (t < my_no) {
                b = bn;
                c = my_val * cn;
                if (b == self) b = -1;  // diagonal: summed above
            }
            if (t + 1 < my_no) {
                bn = idx[(int64_t)my_sig * cap + t + 1];
                cn = (double)val[(int64_t)my_sig * cap + t + 1];
            }
            const bool act = b >= 0;
            const unsigned peers = __match_any_sync(SDB_FULL, act ? b : K + lane);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int gmax = (int)__reduce_max_sync(SDB_FULL, act ? (unsigned)__popc(peers) : 0u);
            for (int r = 0; r < gmax; ++r) {
                if (act && rank == r) row[b] += c;
                __syncwarp();
            }
        }
        __syncwarp();
    }
    if (lane == 0) row[self] += diag;
#pragma unroll
    for (int q = 0; q < MPL; ++q) part[wib][y2 ? 2 * lane + q : lane + 32 * q] = acc[q];
    __syncthreads();
    double* outB = B + e * m;
    for (int r = threadIdx.x; r < m; r += 256) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += part[w][r];
        outB[r] = t;
    }
    double* outA = A + e * K;
    for (int b = threadIdx.x; b < K; b += 256) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += sh_row[(int64_t)w * K + b];
        outA[b] = t;
    }
}

// ---- (f+g), one warp per (shard, atom) bucket: the same two rows as
// k_normal_eq, for launches with enough buckets to fill the GPU with warps
// (P K >= 148 x 32). The warp walks its bucket's 32-entry batches in order
// (four Y rows in flight per batch), keeps its lanes' Y X^T columns in
// registers and its X X^T row in a private shared-memory row, so there is no
// cross-warp combine and no block barrier; the summation order is fixed by
// the bucket order (deterministic).
// a signal's 8 code slots with 16-byte loads (cap == 8: rows are 32 / 64 bytes)
__device__ __forceinline__ void load_row8(const int32_t* __restrict__ p, int (&v)[8]) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p)), b = __ldg(reinterpret_cast<const int4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load_row8(const double* __restrict__ p, double (&v)[8]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p) + q);
        v[2 * q] = a.x;
        v[2 * q + 1] = a.y;
    }
}
__device__ __forceinline__ void load_row8(const float* __restrict__ p, float (&v)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// CAP8 (cap == 8): every entry's index row (the other atoms of its signal) is
// requested with two 16-byte loads before the Y rows are walked, instead of
// one dependent scalar load per (entry, slot) in front of each match.
// Y2 (float rows of exactly 64 values, 8-byte aligned): lane l walks columns
// 2l, 2l + 1 with one 8-byte load per entry (half the load and
// conversion instructions of the lane, lane + 32 walk).
template <typename TY, typename T, int MPL, bool CAP8, bool Y2 = false>
__global__ void __launch_bounds__(256, Y2 ? 4 : (CAP8 && MPL <= 2) ? 4 : 1)
k_normal_eq_w(int64_t PK, int K, int m, const TY* __restrict__ Y, int64_t ldy,
              const int64_t* __restrict__ bucket_off, int cap, const int32_t* __restrict__ idx,
              const T* __restrict__ val, const int32_t* __restrict__ counts, const int32_t* __restrict__ bent,
              double* __restrict__ B, double* __restrict__ A) {
    extern __shared__ double sh_rows[];  // 8 warps x K
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t e = (int64_t)blockIdx.x * 8 + wib;  // (p, a)
    if (e >= PK) return;
    const int self = (int)(e % K);
    double* row = sh_rows + (int64_t)wib * K;
    for (int b = lane; b < K; b += 32) row[b] = 0.0;
    __syncwarp();
    double acc[MPL];
#pragma unroll
    for (int q = 0; q < MPL; ++q) acc[q] = 0.0;
    double diag = 0.0;
    const int64_t lo = bucket_off[e], hi = bucket_off[e + 1];
    for (int64_t b0 = lo; b0 < hi; b0 += 32) {
        const int nbat = (int)min((int64_t)32, hi - b0);
        const int my_e = lane < nbat ? bent[b0 + lane] : 0;
        const int my_sig = my_e / cap;
        const double my_val = lane < nbat ? (double)val[my_e] : 0.0;
        const int my_n = lane < nbat ? counts[my_sig] : 0;
        int bs[8];
        if constexpr (CAP8) {
            if (lane < nbat) {
                load_row8(idx + (int64_t)my_sig * 8, bs);
            } else {
#pragma unroll
                for (int t = 0; t < 8; ++t) bs[t] = -1;
            }
        }
        if constexpr (Y2) {
            for (int j = 0; j < nbat; j += 4) {
                float2 yv[4];
                const bool full = j + 4 <= nbat;   // warp-uniform
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = __shfl_sync(SDB_FULL, my_sig, (j + u) & 31);
                    yv[u] = make_float2(0.f, 0.f);
                    if (full || j + u < nbat)
                        yv[u] = __ldg(reinterpret_cast<const float2*>(Y + (int64_t)i * ldy) + lane);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double v = __shfl_sync(SDB_FULL, my_val, (j + u) & 31);
                    acc[0] = fma((double)yv[u].x, v, acc[0]);
                    acc[1] = fma((double)yv[u].y, v, acc[1]);
                }
            }
        } else
        for (int j = 0; j < nbat; j += 4) {
            double yv[4][MPL];
            double vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = __shfl_sync(SDB_FULL, my_sig, (j + u) & 31);
                vv[u] = __shfl_sync(SDB_FULL, my_val, (j + u) & 31);
                const TY* y = Y + (int64_t)i * ldy;
#pragma unroll
                for (int q = 0; q < MPL; ++q) {
                    const int r = lane + 32 * q;
                    yv[u][q] = (j + u < nbat && r < m) ? (double)y[r] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < MPL; ++q) acc[q] = fma(yv[u][q], vv[u], acc[q]);
        }
        diag += warp_sum(my_val * my_val);
        // the entry's code values: one request for the row instead of a dependent
        // load in front of every slot round
        T vs[8];
        if constexpr (CAP8 && Y2) {
            if (lane < nbat) {
                load_row8(val + (int64_t)my_sig * 8, vs);
            } else {
#pragma unroll
                for (int t = 0; t < 8; ++t) vs[t] = T(0);
            }
        }
        const int my_no = my_n > 1 ? my_n : 0;
        const int nmax = (int)__reduce_max_sync(SDB_FULL, (unsigned)my_no);
        auto slot = [&](int b, double c) {
            if (b == self) b = -1;
            const bool act = b >= 0;
            const unsigned peers = __match_any_sync(SDB_FULL, act ? b : K + lane);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int gmax = (int)__reduce_max_sync(SDB_FULL, act ? (unsigned)__popc(peers) : 0u);
            for (int r = 0; r < gmax; ++r) {
                if (act && rank == r) row[b] += c;
                __syncwarp();
            }
        };
        if constexpr (CAP8) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (t < nmax) {                                  // warp-uniform
                    const bool in = t < my_no;
                    if constexpr (Y2) slot(in ? bs[t] : -1, in ? my_val * (double)vs[t] : 0.0);
                    else slot(in ? bs[t] : -1, in ? my_val * (double)val[(int64_t)my_sig * 8 + t] : 0.0);
                }
            }
        } else {
            for (int t = 0; t < nmax; ++t) {
                int b = -1;
                double c = 0.0;
                if (t < my_no) {
                    b = idx[(int64_t)my_sig * cap + t];
                    c = my_val * (double)val[(int64_t)my_sig * cap + t];
                }
                slot(b, c);
            }
        }
        __syncwarp();
    }
    if (lane == 0) row[self] += diag;
    __syncwarp();
    double* outB = B + e * m;
    if constexpr (Y2) {
        reinterpret_cast<double2*>(outB)[lane] = make_double2(acc[0], acc[1]);
    } else {
#pragma unroll
        for (int q = 0; q < MPL; ++q) {
            const int r = lane + 32 * q;
            if (r < m) outB[r] = acc[q];
        }
    }
    double* outA = A + e * K;
    for (int b = lane; b < K; b += 32) outA[b] = row[b];
}

// ---- per-signal residual ||y_i - D_p x_i||^2 (D in f64, atom-major). With
// `only_if`, shards whose flag is 0 are skipped; if no shard is flagged the
// whole (grid-stride) launch exits after reading the P flags.
template <typename TY, typename T, int MPL>
__global__ void __launch_bounds__(256)
k_resid_sq(int64_t N, int m, int K, int cap, int P, const int64_t* __restrict__ off,
           const TY* __restrict__ Y, int64_t ldy, const int32_t* __restrict__ idx,
           const T* __restrict__ val, const int32_t* __restrict__ counts,
           const double* __restrict__ D, double* __restrict__ out, double* __restrict__ ysq_out,
           const int32_t* __restrict__ only_if) {
    const int lane = threadIdx.x & 31;
    if (only_if) {
        __shared__ int s_any;
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        int any = 0;
        for (int q = threadIdx.x; q < P; q += blockDim.x) any |= only_if[q];
        if (any) s_any = 1;
        __syncthreads();
        if (!s_any) return;
    }
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < N; i += nw) {
        const int p = shard_of(off, P, i);
        if (only_if && only_if[p] == 0) continue;  // warp-uniform
        const double* Dp = D + (int64_t)p * K * m;
        const TY* y = Y + i * ldy;
        double r[MPL];
        double yy = 0.0;
#pragma unroll
        for (int q = 0; q < MPL; ++q) {
            const int row = lane + 32 * q;
            r[q] = (row < m) ? (double)y[row] : 0.0;
            yy = fma(r[q], r[q], yy);
        }
        const int n = counts[i];
        for (int t = 0; t < n; ++t) {
            const double* d = Dp + (int64_t)idx[i * cap + t] * m;
            const double v = (double)val[i * cap + t];
#pragma unroll
            for (int q = 0; q < MPL; ++q) {
                const int row = lane + 32 * q;
                if (row < m) r[q] = fma(-d[row], v, r[q]);
            }
        }
        double sacc = 0.0;
#pragma unroll
        for (int q = 0; q < MPL; ++q) sacc = fma(r[q], r[q], sacc);
        sacc = warp_sum(sacc);
        yy = warp_sum(yy);
        if (lane == 0) {
            out[i] = sacc;
            if (ysq_out) ysq_out[i] = yy;
        }
    }
}

static unsigned resid_grid(int64_t N) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 7) / 8, (int64_t)148 * 16));
}

// ---- ||y_i||^2 per signal
template <typename T, int MPL>
__global__ void __launch_bounds__(256)
k_row_sq(int64_t N, int m, const T* __restrict__ Y, int64_t ldy, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= N) return;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < MPL; ++q) {
        const int r = lane + 32 * q;
        if (r < m) {
            const double v = (double)Y[i * ldy + r];
            s = fma(v, v, s);
        }
    }
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
}

// least-squares residual from the identity; shards whose relative residual^2
// is below 1e-4 (near-exact fits, where the subtraction cancels) are flagged
// for the explicit pass
__global__ void k_ls_resid(int P, const double* __restrict__ ysq, const double* __restrict__ wsq,
                           double* __restrict__ resid, int32_t* __restrict__ need) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const double r2 = ysq[p] - wsq[p];
    resid[p] = sqrt(fmax(r2, 0.0));
    // wsq < 0: minimum-norm fallback solution (no Cholesky identity)
    need[p] = (wsq[p] < 0.0 || r2 <= 1e-4 * ysq[p]) ? 1 : 0;
}

__global__ void __launch_bounds__(256)
k_shard_sum_masked(const int64_t* __restrict__ off, const double* __restrict__ v,
                   const int32_t* __restrict__ mask, double* __restrict__ out) {
    __shared__ double sh[256];
    const int p = blockIdx.x;
    if (!mask[p]) return;
    double s = 0.0;
    for (int64_t i = off[p] + threadIdx.x; i < off[p + 1]; i += 256) s += v[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[p] = sqrt(sh[0]);
}

// ---- deterministic per-shard sum of a per-signal array (fixed order)
__global__ void __launch_bounds__(256)
k_shard_sum(const int64_t* __restrict__ off, const double* __restrict__ v, double* __restrict__ out,
            int do_sqrt) {
    __shared__ double sh[256];
    const int p = blockIdx.x;
    double s = 0.0;
    for (int64_t i = off[p] + threadIdx.x; i < off[p + 1]; i += 256) s += v[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[p] = do_sqrt ? sqrt(sh[0]) : sh[0];
}

// ---- (i) finish MOD: norms, dead atoms, restore, normalise (dictionary_update.py:103-113),
// in two wide launches (warp per atom, 8 atoms per CTA, grid = atom blocks x
// shards): (1) column norms of the raw solution plus per-CTA partials of the
// shard's max norm, used-atom count and code nonzeros; (2) each CTA reduces
// its shard's partials (max / integer sums: order-free) and restores or
// normalises its atoms.
__global__ void __launch_bounds__(256)
k_mod_norms(int P, int K, int m, const double* __restrict__ Z, const int32_t* __restrict__ usage,
            double* __restrict__ scales, double* __restrict__ pmax, int64_t* __restrict__ pnnz,
            int32_t* __restrict__ prank) {
    __shared__ double smx[8];
    __shared__ long long snz[8];
    __shared__ int srk[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int p = blockIdx.y, nb = gridDim.x;
    const int a = blockIdx.x * 8 + wib;
    double nrm = 0.0;
    int u = 0;
    if (a < K) {
        const double* z = Z + ((int64_t)p * K + a) * m;
        double s = 0.0;
        for (int r = lane; r < m; r += 32) s = fma(z[r], z[r], s);
        nrm = sqrt(warp_sum(s));
        u = usage[(int64_t)p * K + a];
        if (lane == 0) scales[(int64_t)p * K + a] = nrm;
    }
    if (lane == 0) { smx[wib] = nrm; snz[wib] = u; srk[wib] = u > 0; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mx = 0.0;
        long long nz = 0;
        int rk = 0;
        for (int w = 0; w < 8; ++w) { mx = fmax(mx, smx[w]); nz += snz[w]; rk += srk[w]; }
        const int64_t q = (int64_t)p * nb + blockIdx.x;
        pmax[q] = mx; pnnz[q] = nz; prank[q] = rk;
    }
}

__global__ void __launch_bounds__(256)
k_mod_apply(int P, int K, int m, const double* __restrict__ Z, const double* __restrict__ Dprev,
            const int32_t* __restrict__ usage, const double* __restrict__ scales, const double* __restrict__ pmax,
            const int64_t* __restrict__ pnnz, const int32_t* __restrict__ prank, int64_t* __restrict__ nnz_shard,
            double* __restrict__ Dout, int8_t* __restrict__ dead, int32_t* __restrict__ rank,
            const int32_t* __restrict__ deficient) {
    __shared__ double s_max;
    __shared__ long long s_nnz;
    __shared__ int s_rank;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int p = blockIdx.y, nb = gridDim.x;
    if (threadIdx.x == 0) {
        double mx = 0.0;
        long long nz = 0;
        int rk = 0;
        for (int b = 0; b < nb; ++b) {
            const int64_t q = (int64_t)p * nb + b;
            mx = fmax(mx, pmax[q]); nz += pnnz[q]; rk += prank[q];
        }
        s_max = mx; s_nnz = nz; s_rank = rk;
        if (blockIdx.x == 0) {
            nnz_shard[p] = nz;
            rank[p] = nz == 0 ? 0 : rk - deficient[p];
        }
    }
    __syncthreads();
    const int a = blockIdx.x * 8 + wib;
    if (a >= K) return;
    const bool empty = s_nnz == 0;
    const double thr = 1e-12 * fmax(s_max, 1.0);
    const int64_t e = (int64_t)p * K + a;
    const bool dd = empty || usage[e] == 0 || scales[e] <= thr;
    if (lane == 0) dead[e] = dd ? 1 : 0;
    const double* src = dd ? (Dprev + e * m) : (Z + e * m);
    double* dst = Dout + e * m;
    if (empty) {  // all-zero codes: D_prev returned unchanged (:92-95)
        for (int r = lane; r < m; r += 32) dst[r] = src[r];
        return;
    }
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(src[r], src[r], s);
    const double nrm = sqrt(warp_sum(s));
    for (int r = lane; r < m; r += 32) dst[r] = nrm > 0.0 ? src[r] / nrm : src[r];
}

// ---- replace_degenerate_atoms (dictionary_update.py:134-176)
// Twin pairs (|<d_a, d_j>| > 0.999 on the normalised atoms, dictionary_update.py:146-151;
// the reference forms the coherences with a BLAS product): a FP32 Gram of the
// FP32-rounded normalised atoms screens the pairs (error ~1e-5, screen at
// 0.998), and only the screened pairs are decided, by the FP64 dot product of
// the FP64 normalised rows (the same routine in both kernels below).
constexpr float TWIN_SCREEN = 0.998f;
__device__ __forceinline__ bool twin_exact(const double* __restrict__ Dn, int64_t ea, int64_t ej, int m, int lane) {
    const double* da = Dn + ea * m;
    const double* dj = Dn + ej * m;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(da[r], dj[r], s);
    return fabs(warp_sum(s)) > 0.999;
}

// (1) warp per (shard, atom): degenerate flag (unused or zero norm) and "row
// has a twin to its right" (j > a);
__global__ void __launch_bounds__(256)
k_twin_flags(int P, int K, const float* __restrict__ C32, const double* __restrict__ Dn,
             const double* __restrict__ D, int m, const int32_t* __restrict__ usage, int8_t* __restrict__ deg,
             int8_t* __restrict__ tw) {
    const int lane = threadIdx.x & 31;
    const int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (e >= (int64_t)P * K) return;
    const int a = (int)(e % K);
    const double* d = D + e * m;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(d[r], d[r], s);
    s = warp_sum(s);
    const float* ci = C32 + e * K;
    bool any = false;
    for (int j0 = a + 1; j0 < K && !any; j0 += 32) {   // warp-uniform
        const int j = j0 + lane;
        unsigned mk = __ballot_sync(SDB_FULL, j < K && fabsf(ci[j]) > TWIN_SCREEN);
        while (mk && !any) {
            const int jj = j0 + __ffs(mk) - 1;
            mk &= mk - 1u;
            any = twin_exact(Dn, e, e - a + jj, m, lane);
        }
    }
    if (lane == 0) {
        deg[e] = (usage[e] == 0 || sqrt(s) <= 1e-12) ? 1 : 0;
        tw[e] = any ? 1 : 0;
    }
}

// (2) one warp per shard: the order-dependent rule (the lower index of a pair
// is kept unless itself degenerate) over the rows that have twins, ascending;
// the columns of a row are screened lane-parallel.
__global__ void __launch_bounds__(32)
k_twins(int K, int m, const float* __restrict__ C32, const double* __restrict__ Dn, const int8_t* __restrict__ tw,
        int8_t* __restrict__ deg, int32_t* __restrict__ ntarget) {
    const int p = blockIdx.x, lane = threadIdx.x;
    const float* Cp = C32 + (int64_t)p * K * K;
    int8_t* dg = deg + (int64_t)p * K;
    const int8_t* twp = tw + (int64_t)p * K;
    for (int i0 = 0; i0 < K; i0 += 32) {
        const unsigned rows = __ballot_sync(SDB_FULL, i0 + lane < K && twp[i0 + lane] != 0);
        for (unsigned r = rows; r; r &= r - 1) {
            const int i = i0 + __ffs(r) - 1;
            __syncwarp();
            if (dg[i]) continue;  // warp-uniform (read after the barrier)
            const float* ci = Cp + (int64_t)i * K;
            for (int j0 = i + 1; j0 < K; j0 += 32) {
                const int j = j0 + lane;
                unsigned mk = __ballot_sync(SDB_FULL, j < K && fabsf(ci[j]) > TWIN_SCREEN);
                while (mk) {
                    const int jj = j0 + __ffs(mk) - 1;
                    mk &= mk - 1u;
                    const bool t = twin_exact(Dn, (int64_t)p * K + i, (int64_t)p * K + jj, m, lane);
                    if (t && lane == 0) dg[jj] = 1;
                }
            }
        }
    }
    __syncwarp();
    int cnt = 0;
    for (int a = lane; a < K; a += 32) cnt += dg[a];
    cnt = __reduce_add_sync(SDB_FULL, cnt);
    if (lane == 0) ntarget[p] = cnt;
}

// normalised copy Dn = D / ||D|| (columns with zero norm untouched)
// (Dn32: optional FP32 rounding of the normalised rows, the twin screen's input)
__global__ void k_normalize_rows(int64_t rows, int m, const double* __restrict__ D, double* __restrict__ Dn,
                                 float* __restrict__ Dn32 = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t a = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (a >= rows) return;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(D[a * m + r], D[a * m + r], s);
    const double nrm = sqrt(warp_sum(s));
    for (int r = lane; r < m; r += 32) {
        const double v = nrm > 0.0 ? D[a * m + r] / nrm : D[a * m + r];
        Dn[a * m + r] = v;
        if (Dn32 != nullptr) Dn32[a * m + r] = (float)v;
    }
}

// Candidate selection: targets (ascending atom) take data columns in order
// of descending residual, ties to the lower column; zero columns skipped.
// One CTA per shard, one block-argmax round per target.
__global__ void __launch_bounds__(512)
k_replace_select(int K, int m, const int64_t* __restrict__ off, const double* __restrict__ rsq,
                 const double* __restrict__ ysq, const int8_t* __restrict__ deg,
                 const int32_t* __restrict__ ntarget, int8_t* __restrict__ taken,
                 int64_t* __restrict__ pick /* P*K: chosen column or -1 */) {
    const int p = blockIdx.x;
    const int64_t lo = off[p], hi = off[p + 1];
    __shared__ double sv[512];
    __shared__ int64_t si[512];
    if (ntarget[p] == 0) return;
    for (int a = 0; a < K; ++a) {
        if (!deg[(int64_t)p * K + a]) continue;
        double bv = -1.0;
        int64_t bi = INT64_MAX;
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            if (taken[i] || !(ysq[i] > 0.0)) continue;
            const double v = rsq[i];
            if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
        sv[threadIdx.x] = bv;
        si[threadIdx.x] = bi;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                const double ov = sv[threadIdx.x + w];
                const int64_t oi = si[threadIdx.x + w];
                if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                    sv[threadIdx.x] = ov;
                    si[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool ok = si[0] != INT64_MAX && sv[0] >= 0.0;
            pick[(int64_t)p * K + a] = ok ? si[0] : -1;
            if (ok) taken[si[0]] = 1;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void k_replace_apply(int P, int K, int m, const T* __restrict__ Y, int64_t ldy,
                                const int8_t* __restrict__ deg, const int64_t* __restrict__ pick,
                                const double* __restrict__ ysq, const int32_t* __restrict__ ntarget,
                                double* __restrict__ D, int8_t* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (e >= (int64_t)P * K) return;
    const int p = (int)(e / K);
    if (ntarget[p] == 0 || !deg[e]) {
        if (lane == 0) flags[e] = 0;
        return;
    }
    const int64_t c = pick[e];
    if (c < 0) {
        if (lane == 0) flags[e] = 2;
        return;
    }
    const double nrm = sqrt(ysq[c]);
    for (int r = lane; r < m; r += 32) D[e * m + r] = (double)Y[c * ldy + r] / nrm;
    if (lane == 0) flags[e] = 1;
}

// ---- usage histogram only (replace_degenerate_atoms called on its own)
__global__ void k_usage_direct(int64_t N, int K, int cap, int P, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ counts,
                               int32_t* __restrict__ usage) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int p = shard_of(off, P, i);
    const int n = counts[i];
    for (int t = 0; t < n; ++t) atomicAdd(&usage[(int64_t)p * K + idx[i * cap + t]], 1);
}


// ---- code energy per shard: sum of squared code values (w_t^2, trainer.py:250)
template <typename T>
__global__ void k_code_sq(int64_t N, int cap, const T* __restrict__ val, const int32_t* __restrict__ counts,
                          double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    double s = 0.0;
    const int n = counts[i];
    for (int t = 0; t < n; ++t) {
        const double v = (double)val[i * cap + t];
        s = fma(v, v, s);
    }
    out[i] = s;
}

// ---- first-columns init per shard (trainer.py:145-148): D0[p][a] =
// normalise(first K signals of shard p); zero columns flagged for the host.
template <typename T>
__global__ void k_first_columns(int P, int K, int m, const int64_t* __restrict__ off,
                                const T* __restrict__ Y, int64_t ldy, double* __restrict__ D,
                                int32_t* __restrict__ zero_flag) {
    const int lane = threadIdx.x & 31;
    const int64_t e = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (e >= (int64_t)P * K) return;
    const int p = (int)(e / K), a = (int)(e % K);
    const T* y = Y + (off[p] + a) * ldy;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma((double)y[r], (double)y[r], s);
    const double nrm = sqrt(warp_sum(s));
    for (int r = lane; r < m; r += 32) D[e * m + r] = nrm > 0.0 ? (double)y[r] / nrm : 0.0;
    if (lane == 0) zero_flag[e] = nrm > 0.0 ? 0 : 1;
}

// ---- merge dataset rows: out[t*K1 + a] = w_t * D_t[a]  (trainer.py:248-256)
template <typename T>
__global__ void k_scale_rows(int64_t rows, int group, int m, const double* __restrict__ D,
                             const double* __restrict__ w, T* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * m) return;
    const int64_t row = e / m;
    out[e] = (T)(w[row / group] * D[e]);
}

// =============================================================================
// host launchers
// =============================================================================
template <typename F>
static int with_mpl(int m, F&& f) {
    const int mpl = (m + 31) / 32;
    if (mpl <= 1) return f(std::integral_constant<int, 1>{});
    if (mpl <= 2) return f(std::integral_constant<int, 2>{});
    if (mpl <= 4) return f(std::integral_constant<int, 4>{});
    if (mpl <= 8) return f(std::integral_constant<int, 8>{});
    return (int)cudaErrorInvalidValue;  // m > 256 rejected at the ABI
}

static int64_t nchunks_upper(int64_t N, int P) { return N / chunk_size(N) + P + 1; }

ModWs carve_mod_ws(void* base, int P, int64_t N, int m, int K, int cap) {
    ModWs w{};
    unsigned char* p = (unsigned char*)base;
    auto take = [&](int64_t bytes) { void* r = p; p += (bytes + 255) & ~int64_t(255); return r; };
    const int64_t nch = nchunks_upper(N, P);
    w.cf = (int64_t*)take(sizeof(int64_t) * (P + 1));
    w.chunk_hist = (int32_t*)take(sizeof(int32_t) * nch * K);
    w.chunk_off = (int64_t*)take(sizeof(int64_t) * nch * K);
    w.wpart = (int64_t*)take(sizeof(int64_t) * SCW * (int64_t)P * K);
    w.bucket_off = (int64_t*)take(sizeof(int64_t) * ((int64_t)P * K + 1));
    w.scan_ws = (int64_t*)take(scan_workspace_bytes((int64_t)P * K));
    w.bent = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(N * cap, 1));
    w.A = (double*)take(sizeof(double) * (int64_t)P * K * K);
    w.B = (double*)take(sizeof(double) * (int64_t)P * K * m);
    w.rsq = (double*)take(sizeof(double) * std::max<int64_t>(N, 1));
    w.nnz = (int64_t*)take(sizeof(int64_t) * P);
    {
        const int64_t nbp = (int64_t)P * ((K + 7) / 8);  // per-CTA partials of the MOD finish
        w.fmax = (double*)take(sizeof(double) * nbp);
        w.fnnz = (int64_t*)take(sizeof(int64_t) * nbp);
        w.frank = (int32_t*)take(sizeof(int32_t) * nbp);
    }
    w.deficient = (int32_t*)take(sizeof(int32_t) * P);
    w.depmask = (int8_t*)take((int64_t)P * K);
    w.chol = take(chol_ws_bytes(P, K));
    w.wsq = (double*)take(sizeof(double) * P);
    w.ysqp = (double*)take(sizeof(double) * P);
    w.need = (int32_t*)take(sizeof(int32_t) * P);
    w.mn = (double*)take(minnorm_ws_bytes(P, m, K));
    w.end = p;
    return w;
}

int64_t mod_ws_bytes(int P, int64_t N, int m, int K, int cap) {
    ModWs w = carve_mod_ws(nullptr, P, N, m, K, cap);
    return (int64_t)(w.end - (unsigned char*)nullptr) + 256;
}

// TY: the signal rows' type (float rows with FP64 codes in the certified
// FP32 mode: the values are exactly the FP64 copy's, at half the gather bytes)
template <typename TY, typename T>
static int mod_update_impl(const ModArgs<T>& a, const TY* Ysrc, cudaStream_t st) {
    const int P = a.P, K = a.K, m = a.m, cap = a.cap;
    const int64_t N = a.N;
    ModWs w = carve_mod_ws(a.ws, P, N, m, K, cap);
    const int64_t PK = (int64_t)P * K;
    const int64_t nch_max = nchunks_upper(N, P);
    const int ch = chunk_size(N);
    k_chunk_layout<<<1, 32, 0, st>>>(a.off, P, ch, w.cf);
    const unsigned hb = (unsigned)((nch_max + 7) / 8);
    k_chunk_hist<<<(unsigned)nch_max, std::min(256, std::max(32, ch)), K * sizeof(int32_t), st>>>(
        a.off, w.cf, P, K, cap, ch, a.idx, a.counts, w.chunk_hist);
    const dim3 gpk((unsigned)((K + 31) / 32), (unsigned)P);
    k_usage_from_chunks<<<gpk, SCW * 32, 0, st>>>(w.cf, P, K, w.chunk_hist, w.wpart, a.usage);
    int rc = exclusive_scan_counts(a.usage, PK, w.bucket_off, w.scan_ws, st);
    if (rc) return rc;
    k_chunk_offsets<<<gpk, SCW * 32, 0, st>>>(w.cf, P, K, w.chunk_hist, w.wpart, w.bucket_off, w.chunk_off);
    {
        const int smem = 8 * K * (int)sizeof(int64_t);
        if (smem > 48 * 1024) {
            cudaError_t e = set_max_smem((const void*)k_place<T>, smem);
            if (e != cudaSuccess) return (int)e;
        }
        k_place<T><<<hb, 256, smem, st>>>(a.off, w.cf, P, K, cap, ch, a.idx, a.val, a.counts,
                                         w.chunk_off, w.bent);
    }
    rc = with_mpl(m, [&](auto c) {
        constexpr int MPL = decltype(c)::value;
        if (PK >= (int64_t)148 * 32) {
            // enough buckets for a warp each
            const int smem = 8 * K * (int)sizeof(double);
            const bool cap8 = cap == 8 && (reinterpret_cast<uintptr_t>(a.idx) & 15) == 0 &&
                              (reinterpret_cast<uintptr_t>(a.val) & 15) == 0;
            auto go = [&](auto kern) -> int {
                if (smem > 48 * 1024) {
                    cudaError_t e = set_max_smem((const void*)kern, smem);
                    if (e != cudaSuccess) return (int)e;
                }
                kern<<<(unsigned)((PK + 7) / 8), 256, smem, st>>>(PK, K, m, Ysrc, a.ldy, w.bucket_off, cap, a.idx,
                                                                 a.val, a.counts, w.bent, w.B, w.A);
                return (int)cudaGetLastError();
            };
            if constexpr (std::is_same<TY, float>::value && MPL == 2) {
                if (cap8 && m == 64 && (a.ldy & 1) == 0 && (reinterpret_cast<uintptr_t>(Ysrc) & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(w.B) & 15) == 0)
                    return go(k_normal_eq_w<TY, T, MPL, true, true>);
            }
            return cap8 ? go(k_normal_eq_w<TY, T, MPL, true>) : go(k_normal_eq_w<TY, T, MPL, false>);
        }
        const int smem = 8 * (K + 32 * MPL) * (int)sizeof(double);
        if (smem > 48 * 1024) {
            cudaError_t e = set_max_smem((const void*)k_normal_eq<TY, T, MPL>, smem);
            if (e != cudaSuccess) return (int)e;
        }
        k_normal_eq<TY, T, MPL><<<(unsigned)PK, 256, smem, st>>>(P, K, m, Ysrc, a.ldy, w.bucket_off, cap, a.idx,
                                                             a.val, a.counts, w.bent, w.B, w.A);
        return (int)cudaGetLastError();
    });
    if (rc) return rc;
    // masked RHS rows of unused atoms are irrelevant: A is the identity there
    // and B holds zeros (their buckets are empty).
    // the Cholesky flags shards with a (near-)dependent pivot; those get the
    // reference's minimum-norm lstsq solution (rank rule rcond) instead
    rc = chol_solve(P, K, m, w.A, w.B, a.usage, std::max(a.rank_rcond, MN_FLAG_TOL), w.depmask, w.deficient,
                    w.wsq, w.chol, st);
    if (rc) return rc;
    rc = minnorm_solve<TY, T>(P, K, m, Ysrc, a.ldy, cap, a.idx, a.val, a.counts, w.bucket_off, w.bent, a.usage,
                          a.rank_rcond, w.A, w.B, w.deficient, w.wsq, w.mn, st);
    if (rc) return rc;
    // residual before normalisation: ||Y - Z^T X||^2 = ||Y||^2 - <Z, B> and
    // <Z, B> = ||L^-1 B||^2 (captured between the forward and back phases)
    const double* ysq = a.ysq_shard;
    if (ysq == nullptr) {
        rc = with_mpl(m, [&](auto c) {
            constexpr int MPL = decltype(c)::value;
            k_row_sq<TY, MPL><<<(unsigned)((N + 7) / 8), 256, 0, st>>>(N, m, Ysrc, a.ldy, w.rsq);
            return (int)cudaGetLastError();
        });
        if (rc) return rc;
        k_shard_sum<<<P, 256, 0, st>>>(a.off, w.rsq, w.ysqp, 0);
        ysq = w.ysqp;
    }
    k_ls_resid<<<(P + 127) / 128, 128, 0, st>>>(P, ysq, w.wsq, a.resid_fro, w.need);
    rc = with_mpl(m, [&](auto c) {
        constexpr int MPL = decltype(c)::value;
        k_resid_sq<TY, T, MPL><<<resid_grid(N), 256, 0, st>>>(
            N, m, K, cap, P, a.off, Ysrc, a.ldy, a.idx, a.val, a.counts, w.B, w.rsq, nullptr, w.need);
        return (int)cudaGetLastError();
    });
    if (rc) return rc;
    k_shard_sum_masked<<<P, 256, 0, st>>>(a.off, w.rsq, w.need, a.resid_fro);
    {
        const dim3 g((unsigned)((K + 7) / 8), (unsigned)P);
        k_mod_norms<<<g, 256, 0, st>>>(P, K, m, w.B, a.usage, a.scales, w.fmax, w.fnnz, w.frank);
        k_mod_apply<<<g, 256, 0, st>>>(P, K, m, w.B, a.Dprev, a.usage, a.scales, w.fmax, w.fnnz, w.frank,
                                       w.nnz, a.Dout, a.dead, a.rank, w.deficient);
    }
    if (a.deficient_out)
        cudaMemcpyAsync(a.deficient_out, w.deficient, sizeof(int32_t) * P, cudaMemcpyDeviceToDevice, st);
    if (a.nnz_out)
        cudaMemcpyAsync(a.nnz_out, w.nnz, sizeof(int64_t) * P, cudaMemcpyDeviceToDevice, st);
    return (int)cudaGetLastError();
}
template <typename T>
int mod_update(const ModArgs<T>& a, cudaStream_t st) {
    if constexpr (std::is_same_v<T, double>) {
        if (a.Yf != nullptr) return mod_update_impl<float, double>(a, a.Yf, st);
    }
    return mod_update_impl<T, T>(a, a.Y, st);
}
template int mod_update<float>(const ModArgs<float>&, cudaStream_t);
template int mod_update<double>(const ModArgs<double>&, cudaStream_t);

int64_t replace_ws_bytes(int P, int64_t N, int m, int K) {
    int64_t b = 0;
    auto add = [&](int64_t x) { b += (x + 255) & ~int64_t(255); };
    add(sizeof(double) * (int64_t)P * K * m);  // normalised copy
    add(sizeof(double) * (int64_t)P * K * K);  // |Dn^T Dn|
    add(sizeof(int8_t) * (int64_t)P * K);      // degenerate flags
    add(sizeof(int8_t) * (int64_t)P * K);      // twin flags
    add(sizeof(int32_t) * P);                  // targets per shard
    add(sizeof(double) * std::max<int64_t>(N, 1));  // residual^2
    add(sizeof(double) * std::max<int64_t>(N, 1));  // ||y||^2
    add(sizeof(int8_t) * std::max<int64_t>(N, 1));  // taken
    add(sizeof(int64_t) * (int64_t)P * K);     // picks
    add(sizeof(float) * (int64_t)P * K * m);   // FP32 normalised copy (twin screen)
    return b + 256;
}

template <typename T>
int replace_degenerate(const ReplaceArgs<T>& a, cudaStream_t st) {
    const int P = a.P, K = a.K, m = a.m, cap = a.cap;
    const int64_t N = a.N, PK = (int64_t)P * K;
    unsigned char* p = (unsigned char*)a.ws;
    auto take = [&](int64_t bytes) { void* r = p; p += (bytes + 255) & ~int64_t(255); return r; };
    double* Dn = (double*)take(sizeof(double) * PK * m);
    float* C32 = (float*)take(sizeof(double) * PK * K);   // FP32 coherence screen (half the slot)
    int8_t* deg = (int8_t*)take(PK);
    int8_t* twin = (int8_t*)take(PK);
    int32_t* ntarget = (int32_t*)take(sizeof(int32_t) * P);
    double* rsq = (double*)take(sizeof(double) * std::max<int64_t>(N, 1));
    double* ysq = (double*)take(sizeof(double) * std::max<int64_t>(N, 1));
    int8_t* taken = (int8_t*)take(std::max<int64_t>(N, 1));
    int64_t* pick = (int64_t*)take(sizeof(int64_t) * PK);
    float* Dn32 = (float*)take(sizeof(float) * PK * m);

    k_normalize_rows<<<(unsigned)((PK + 7) / 8), 256, 0, st>>>(PK, m, a.D, Dn, Dn32);
    int rc = gram_screen_f32(Dn32, P, m, K, C32, st);
    if (rc) return rc;
    k_twin_flags<<<(unsigned)((PK + 7) / 8), 256, 0, st>>>(P, K, C32, Dn, a.D, m, a.usage, deg, twin);
    k_twins<<<P, 32, 0, st>>>(K, m, C32, Dn, twin, deg, ntarget);
    // residuals with the current D and the given codes (always computed; the
    // reference skips them when no atom is degenerate, which changes nothing)
    rc = with_mpl(m, [&](auto c) {
        constexpr int MPL = decltype(c)::value;
        k_resid_sq<T, T, MPL><<<resid_grid(N), 256, 0, st>>>(
            N, m, K, cap, P, a.off, a.Y, a.ldy, a.idx, a.val, a.counts, a.D, rsq, ysq, ntarget);
        return (int)cudaGetLastError();
    });
    if (rc) return rc;
    if (N > 0) cudaMemsetAsync(taken, 0, N, st);
    k_replace_select<<<P, 512, 0, st>>>(K, m, a.off, rsq, ysq, deg, ntarget, taken, pick);
    k_replace_apply<T><<<(unsigned)((PK + 7) / 8), 256, 0, st>>>(P, K, m, a.Y, a.ldy, deg, pick, ysq,
                                                                ntarget, a.D, a.flags);
    if (a.ntarget_out)
        cudaMemcpyAsync(a.ntarget_out, ntarget, sizeof(int32_t) * P, cudaMemcpyDeviceToDevice, st);
    return (int)cudaGetLastError();
}
template int replace_degenerate<float>(const ReplaceArgs<float>&, cudaStream_t);
template int replace_degenerate<double>(const ReplaceArgs<double>&, cudaStream_t);

template <typename T>
int residual_sq(int64_t N, int m, int K, int cap, int P, const int64_t* off, const T* Y, int64_t ldy,
                const int32_t* idx, const T* val, const int32_t* counts, const double* D,
                double* rsq, double* ysq, cudaStream_t st) {
    if (N <= 0) return 0;
    return with_mpl(m, [&](auto c) {
        constexpr int MPL = decltype(c)::value;
        k_resid_sq<T, T, MPL><<<resid_grid(N), 256, 0, st>>>(N, m, K, cap, P, off, Y, ldy, idx,
                                                                   val, counts, D, rsq, ysq, nullptr);
        return (int)cudaGetLastError();
    });
}
template int residual_sq<float>(int64_t, int, int, int, int, const int64_t*, const float*, int64_t,
                                const int32_t*, const float*, const int32_t*, const double*, double*,
                                double*, cudaStream_t);
template int residual_sq<double>(int64_t, int, int, int, int, const int64_t*, const double*, int64_t,
                                 const int32_t*, const double*, const int32_t*, const double*, double*,
                                 double*, cudaStream_t);

int shard_ysq(int P, int64_t N, int m, const void* Y, int64_t ldy, bool f64, const int64_t* off,
              double* tmp, double* out, cudaStream_t st) {
    if (N > 0) {
        int rc = with_mpl(m, [&](auto c) {
            constexpr int MPL = decltype(c)::value;
            if (f64)
                k_row_sq<double, MPL><<<(unsigned)((N + 7) / 8), 256, 0, st>>>(N, m, (const double*)Y, ldy, tmp);
            else
                k_row_sq<float, MPL><<<(unsigned)((N + 7) / 8), 256, 0, st>>>(N, m, (const float*)Y, ldy, tmp);
            return (int)cudaGetLastError();
        });
        if (rc) return rc;
    }
    k_shard_sum<<<P, 256, 0, st>>>(off, tmp, out, 0);
    return (int)cudaGetLastError();
}

int shard_sum(int P, const int64_t* off, const double* v, double* out, int do_sqrt, cudaStream_t st) {
    k_shard_sum<<<P, 256, 0, st>>>(off, v, out, do_sqrt);
    return (int)cudaGetLastError();
}

int usage_direct(int64_t N, int K, int cap, int P, const int64_t* off, const int32_t* idx,
                 const int32_t* counts, int32_t* usage, cudaStream_t st) {
    cudaMemsetAsync(usage, 0, sizeof(int32_t) * (int64_t)P * K, st);
    if (N > 0)
        k_usage_direct<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, K, cap, P, off, idx, counts, usage);
    return (int)cudaGetLastError();
}

template <typename T>
int code_sq(int64_t N, int cap, const T* val, const int32_t* counts, double* out, cudaStream_t st) {
    if (N <= 0) return 0;
    k_code_sq<T><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, cap, val, counts, out);
    return (int)cudaGetLastError();
}
template int code_sq<float>(int64_t, int, const float*, const int32_t*, double*, cudaStream_t);
template int code_sq<double>(int64_t, int, const double*, const int32_t*, double*, cudaStream_t);

template <typename T>
int first_columns(int P, int K, int m, const int64_t* off, const T* Y, int64_t ldy, double* D,
                  int32_t* zero_flag, cudaStream_t st) {
    const int64_t PK = (int64_t)P * K;
    k_first_columns<T><<<(unsigned)((PK + 7) / 8), 256, 0, st>>>(P, K, m, off, Y, ldy, D, zero_flag);
    return (int)cudaGetLastError();
}
template int first_columns<float>(int, int, int, const int64_t*, const float*, int64_t, double*, int32_t*, cudaStream_t);
template int first_columns<double>(int, int, int, const int64_t*, const double*, int64_t, double*, int32_t*, cudaStream_t);

template <typename T>
int scale_rows(int64_t rows, int group, int m, const double* D, const double* w, T* out, cudaStream_t st) {
    const int64_t n = rows * m;
    if (n <= 0) return 0;
    k_scale_rows<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rows, group, m, D, w, out);
    return (int)cudaGetLastError();
}
template int scale_rows<float>(int64_t, int, int, const double*, const double*, float*, cudaStream_t);
template int scale_rows<double>(int64_t, int, int, const double*, const double*, double*, cudaStream_t);

}  // namespace sdb
