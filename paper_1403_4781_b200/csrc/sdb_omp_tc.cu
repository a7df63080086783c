// Fused tensor-core Batch-OMP (FP32 mode, sm_100a): omp_single
// (_kernels.py:38-158) for tiles of 128 signals of one shard, where every
// greedy step's correlations corr = D^T r are ONE tcgen05 MMA of the tile's
// residual matrix R (128 x m, shared memory) against the shard's dictionary
// (K x m, resident in shared memory) into TMEM — the alpha0 = D^T Y GEMM is the
// first step's MMA, so no correlation matrix ever touches HBM and no G row is
// streamed per step (the Batch-OMP update corr = c0 - G_S x of k_omp_fast is
// replaced by recomputing D^T r on the tensor pipe).
//
// Precision. The MMA is kind::tf32 (operands truncated to 10-bit mantissas,
// fp32 accumulation), so |corr_tf32 - d.r| <= 2^-9 ||d|| ||r|| (+ 2^-16 ||r||
// accumulation). The argmax is decided exactly: every atom whose TF32 value
// lies within a window (2^-8 ||r||, twice the bound, plus 1e-6 ||y|| for the
// numerical residue of support atoms) of the TF32 maximum is a candidate, and
// the candidates' correlations are recomputed in FP32 on the CUDA cores from
// the resident dictionary and the exact residual (both in shared memory);
// the largest |d.r| wins, lowest index on ties (the reference's 1e-12 tie
// window is below FP32 resolution, as in k_omp_fast). More than OT_CMAX
// candidates (or none outside the support) fall back to an exact sweep over
// all atoms. Per signal the smallest decision margin is reported (near-tie
// log, north_star; the FP64 certification pass re-decides signals whose
// margin is below its tolerance, sdb_certify.cu): over the steps whose best
// |d.r| is above the rounding floor (1e-6 ||y||), (best - runner-up) / ||y||
// with the runner-up exact among the candidates and bounded above by
// thr + win/2 for the rest; and in error-bounded mode |(||r|| - eps)| / ||y||
// at every stopping test.
//
// Per step and signal (thread = signal, TMEM lane = tile row):
//   scan:   block maxima of |corr_tf32| over the row (tcgen05.ld), then the
//           candidates above the threshold (second TMEM pass on the blocks
//           some lane needs)
//   refine: exact d_j.r for the candidates (shared memory)
//   stop:   stall (cmax <= 1e-13 ||r||, _kernels.py:97-100); Cholesky append
//           with G[S,b], G[b,b] (L2) and the singular guard (_kernels.py:109-127)
//   solve:  forward/back substitution with L in registers (_kernels.py:129-139)
//   update: r -= D_S (x_new - x_old) in place in R (the next MMA's A operand),
//           ||r||^2 explicit (_kernels.py:141-154); eps test on ||r||
//
// Roles (one persistent CTA per SM, 10 warps):
//   warp 0    TMA producer: the shard's padded dictionary (4 boxes of 256 x 32)
//   warp 1    TMEM allocation (512 columns) + MMA issuer (one thread)
//   warps 2-5 signal group 0, warps 6-9 signal group 1: each group codes its
//             own tile; the MMA of one group's step overlaps the other
//             group's CUDA-core work. K > 256: the two 256-column chunk
//             buffers alternate between the groups; K <= 256: one buffer each.
// Tiles: each CTA owns a contiguous range of the (shard, tile) sequence and
// walks it in rounds of two tiles of the same shard; the dictionary is
// reloaded when the shard changes (after both groups released the old one).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_tc.cuh"

namespace sdb {

bool tc_map_f32(CUtensorMap* map, const float* ptr, int64_t cols, int64_t rows, int64_t ld_elems,
                int box_rows);

namespace {

constexpr int OT_M = 128;          // signals per tile (UMMA M, TMEM lanes)
constexpr int OT_N = 256;          // atoms per MMA chunk (UMMA N)
constexpr int OT_NGMAX = 3;        // signal groups (tiles in flight per CTA): 2, or 3 when K > 256
constexpr int OT_CMAX = 6;         // candidates refined per step before the exact sweep
constexpr float OT_WIN = 0.00390625f;   // 2^-8: candidate window, relative to ||r||
constexpr int OT_RB = OT_M * 128;  // bytes of one 32-column k-block of R

struct OtArgs {
    int64_t N;
    int m, K, P, cap, nkb, nch, kpad, clen;
    const int64_t* off;   // P+1 signal offsets
    const int64_t* ts;    // P+1 tile prefix (first tile of each shard)
    const float* Y;
    int64_t ldy;
    const float* G;       // P x K x K
    float eps, guard;
    int32_t* idx;
    float* val;
    int32_t* counts;
    int8_t* status;
    float* rnorm;         // optional
    float* gap;           // optional: smallest decision margin / ||y|| over the steps
};

__device__ __forceinline__ int tile_shard(const int64_t* __restrict__ ts, int P, int64_t t) {
    int lo = 0, hi = P - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(ts + mid) <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// A round: up to NG consecutive tiles of one shard (one per signal group).
struct Round {
    int p;
    int64_t t0;
    int cnt;            // tiles in this round (1..NG), one per signal group
    bool first, last;   // the CTA's first / last round on this shard's dictionary
};

// The (shard, tile) sequence is cut into chunks of `clen` consecutive tiles,
// dealt round-robin to the CTAs: at any time the grid works on ~grid * clen
// consecutive tiles (a few shards), so the Gram rows the Cholesky appends
// gather stay in L2 (a contiguous range per CTA had ~100 shards' Gram matrices
// live at once: 5.6 GB of HBM sector reads per C4 pass). Within a chunk the
// shard index advances linearly; one binary search per chunk.
template <int NG>
struct RoundIter {
    const int64_t* ts;
    int P, clen;
    int64_t ntiles, cnext, cstride;
    int64_t pos, cend, pend;
    int p, prev, pnext;
    __device__ RoundIter(const int64_t* ts_, int P_, int clen_)
        : ts(ts_), P(P_), clen(clen_), pos(0), cend(0), pend(0), p(0), prev(-1) {
        ntiles = __ldg(ts + P);
        cnext = (int64_t)blockIdx.x * clen;
        cstride = (int64_t)gridDim.x * clen;
        pnext = cnext < ntiles ? tile_shard(ts, P, cnext) : -1;
    }
    __device__ bool next(Round& r) {
        if (pos >= cend) {
            if (cnext >= ntiles) return false;
            pos = cnext;
            cend = min(ntiles, cnext + clen);
            p = pnext;
            pend = __ldg(ts + p + 1);
            cnext += cstride;
            pnext = cnext < ntiles ? tile_shard(ts, P, cnext) : -1;
        } else {
            while (pos >= pend) {   // next shard (empty shards own no tiles)
                ++p;
                pend = __ldg(ts + p + 1);
            }
        }
        r.p = p;
        r.t0 = pos;
        const int64_t lim = min(cend, pend);
        r.cnt = (int)min((int64_t)NG, lim - pos);
        pos += r.cnt;
        r.first = p != prev;
        prev = p;
        // the dictionary is released when the CTA's next round is on another shard
        r.last = pos >= cend ? (pnext != p) : (pos >= pend);
        return true;
    }
};


// CAP: code slots; NG: signal groups; NKB: 32-column k-blocks of m (m_pad / 32);
// NCH: 256-atom chunks of K
template <int CAP, int NG, int NKB, int NCH>
__global__ void __launch_bounds__((2 + 4 * NG) * 32, 1)
k_omp_tc(const __grid_constant__ CUtensorMap tmD, const OtArgs a) {
    constexpr int KPAD = NCH * OT_N;
    // barriers: full[g] (MMA done / tile end ack), empty[b] (TMEM chunk buffer
    // free), rfull[g] (residual published), dfull (dictionary landed), dfree
    constexpr int B_FULL = 0, B_EMPTY = NG, B_RFULL = NG + 2, B_DFULL = 2 * NG + 2, B_DFREE = 2 * NG + 3;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr int dbytes = NKB * KPAD * 128;
    constexpr int rbytes = NKB * OT_RB;
    unsigned char* Ds = base;
    // per-lane slots (128 B: the block of the running maximum; chunk-major, 16 B
    // of every lane side by side), then the barriers
    unsigned char* Sl = base + dbytes + NG * rbytes;
    uint64_t* bars = (uint64_t*)(Sl + NG * OT_M * 128);
    int* votes = (int*)(bars + 2 * NG + 4);   // [step parity][group][warp]
    volatile int* contf = votes + 8 * NG;     // [group]
    uint32_t* tslot = (uint32_t*)(votes + 9 * NG);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K = a.K;

    if (threadIdx.x == 0) {
        for (int g = 0; g < NG; ++g) {
            mbar_init(smem_u32(&bars[B_FULL + g]), 1);
            mbar_init(smem_u32(&bars[B_RFULL + g]), 4);
        }
        for (int b = 0; b < 2; ++b) mbar_init(smem_u32(&bars[B_EMPTY + b]), 4);
        mbar_init(smem_u32(&bars[B_DFULL]), 1);
        mbar_init(smem_u32(&bars[B_DFREE]), 4 * NG);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(2 * OT_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // ------------------------------------------------ dictionary producer
        if (lane == 0) {
            RoundIter<NG> it(a.ts, a.P, a.clen);
            Round r;
            int k = 0;
            while (it.next(r)) {
                if (!r.first) continue;
                if (k > 0) mbar_wait_sleep(smem_u32(&bars[B_DFREE]), (uint32_t)((k - 1) & 1));
                const uint32_t bf = smem_u32(&bars[B_DFULL]);
                mbar_expect_tx(bf, (uint32_t)dbytes);
                for (int kb = 0; kb < NKB; ++kb)
                    for (int c = 0; c < NCH; ++c)
                        tma_load_2d(smem_u32(Ds + kb * KPAD * 128 + c * OT_N * 128), &tmD, kb * 32,
                                    r.p * KPAD + c * OT_N, bf);
                ++k;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(OT_N >> 3) << 17) |
                                   ((uint32_t)(OT_M >> 4) << 24);
            uint32_t uses[2] = {0, 0}, rph[NG];
            for (int g = 0; g < NG; ++g) rph[g] = 0;
            int k = 0;
            RoundIter<NG> it(a.ts, a.P, a.clen);
            Round r;
            while (it.next(r)) {
                if (r.first) {
                    mbar_wait_sleep(smem_u32(&bars[B_DFULL]), (uint32_t)(k & 1));
                    ++k;
                }
                bool act[NG];
                int nact = r.cnt;
                for (int g = 0; g < NG; ++g) act[g] = g < r.cnt;
                while (nact > 0) {
                    for (int g = 0; g < NG; ++g) {
                        if (!act[g]) continue;
                        mbar_wait_sleep(smem_u32(&bars[B_RFULL + g]), rph[g] & 1u);
                        ++rph[g];
                        if (!contf[g]) {
                            // tile done: acknowledge on full[g] so the group cannot
                            // publish its next tile before this phase was consumed
                            mbar_arrive(smem_u32(&bars[B_FULL + g]));
                            act[g] = false;
                            --nact;
                            continue;
                        }
                        const unsigned char* Rg = base + dbytes + g * rbytes;
                        for (int c = 0; c < NCH; ++c) {
                            const int b = NCH == 2 ? c : (g & 1);
                            if (uses[b]) mbar_wait_sleep(smem_u32(&bars[B_EMPTY + b]), (uses[b] - 1) & 1u);
                            ++uses[b];
                            tmem_fence_after();
                            const uint32_t tacc = tmem + (uint32_t)(b * OT_N);
                            for (int kb = 0; kb < NKB; ++kb) {
                                const uint64_t ad = sw128_desc(smem_u32(Rg + kb * OT_RB));
                                const uint64_t bd = sw128_desc(smem_u32(Ds + kb * KPAD * 128 + c * OT_N * 128));
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    mma_tf32(tacc, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc,
                                             (kb | kk) ? 1u : 0u);
                            }
                        }
                        mma_commit(smem_u32(&bars[B_FULL + g]));
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ signal groups
        const int g = (warp - 2) >> 2;
        const int wi = (warp - 2) & 3;
        const int q = warp & 3;                 // TMEM lane quadrant of this warp
        const int row = q * 32 + lane;          // tile row = TMEM lane
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        // shared-space addresses: the lane's residual row (chunk cc of k-block kb at
        // (rpre ^ (cc << 4)) + kb * OT_RB, 128-byte swizzle) and slot
        const uint32_t ds_u32 = smem_u32(Ds);
        const uint32_t rpre = (smem_u32(base + dbytes + g * rbytes) + (uint32_t)row * 128u) ^ ((uint32_t)(row & 7) << 4);
        const uint32_t slot = smem_u32(Sl) + (uint32_t)(g * OT_M * 128 + row * 16);
        uint32_t fph = 0;
        int sp = 0;
        int k = 0;
        RoundIter<NG> it(a.ts, a.P, a.clen);
        Round rd;
        // atom j's dictionary row: chunk cc of k-block kb at (dpre(j) ^ (cc << 4)) + kb * KPAD * 128
        auto dpre = [&](int j) -> uint32_t { return (ds_u32 + ((uint32_t)j << 7)) ^ (((uint32_t)j & 7u) << 4); };
        // d_j . r (exact FP32, both operands in shared memory)
        auto dot = [&](int j) -> float {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
            const uint32_t dp = dpre(j);
#pragma unroll
            for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const float4 d = lds4_u32((dp ^ (uint32_t)(cc << 4)) + (uint32_t)(kb * KPAD * 128));
                    const float4 v = lds4_u32((rpre ^ (uint32_t)(cc << 4)) + (uint32_t)(kb * OT_RB));
                    s0 = fmaf(d.x, v.x, s0);
                    s1 = fmaf(d.y, v.y, s1);
                    s2 = fmaf(d.z, v.z, s2);
                    s3 = fmaf(d.w, v.w, s3);
                }
            }
            return (s0 + s1) + (s2 + s3);
        };
        // votes of the group's four warps -> 1 if any lane wants another MMA
        auto publish = [&](bool want) -> int {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // R writes -> MMA (async proxy)
            const unsigned bal = __ballot_sync(SDB_FULL, want);
            int* vs = votes + (sp * NG + g) * 4;
            if (lane == 0) vs[wi] = bal != 0u;
            asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
            const int c = vs[0] | vs[1] | vs[2] | vs[3];
            sp ^= 1;
            __syncwarp();
            if (lane == 0) {
                if (wi == 0) contf[g] = c;
                mbar_arrive(smem_u32(&bars[B_RFULL + g]));
            }
            return c;
        };

        while (it.next(rd)) {
            if (rd.first) {
                mbar_wait_sleep(smem_u32(&bars[B_DFULL]), (uint32_t)(k & 1));   // the shard's dictionary landed
                ++k;
            }
            if (g < rd.cnt) {
                const int p = rd.p;
                const int64_t tile = rd.t0 + g;
                const int64_t row0 = __ldg(a.off + p) + (tile - __ldg(a.ts + p)) * OT_M;
                const int64_t i = row0 + row;
                const bool valid = i < __ldg(a.off + p + 1);
                const float* __restrict__ Gp = a.G + (int64_t)p * K * K;
                // ---- the tile's signals -> R (the first step's A operand), ||y||^2
                float ysq = 0.0f;
                {
                    const float* yr = a.Y + i * a.ldy;
                    // the group's next tile (normally NG tiles on) is pulled into L2
                    // while this one is coded
                    {
                        const int64_t inext = i + (int64_t)NG * OT_M;
                        if (inext < a.N) {
                            const float* yn = a.Y + inext * a.ldy;
                            for (int c = 0; c < a.m; c += 32)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(yn + c));
                        }
                    }
                    const bool vec = ((a.ldy & 3) == 0) && ((((uintptr_t)a.Y) & 15) == 0);
#pragma unroll
                    for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc) {
                            const int col = kb * 32 + cc * 4;
                            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (valid) {
                                if (vec && col + 3 < a.m) {
                                    v = __ldg(reinterpret_cast<const float4*>(yr + col));
                                } else {
                                    if (col < a.m) v.x = __ldg(yr + col);
                                    if (col + 1 < a.m) v.y = __ldg(yr + col + 1);
                                    if (col + 2 < a.m) v.z = __ldg(yr + col + 2);
                                    if (col + 3 < a.m) v.w = __ldg(yr + col + 3);
                                }
                            }
                            ysq = fmaf(v.x, v.x, ysq);
                            ysq = fmaf(v.y, v.y, ysq);
                            ysq = fmaf(v.z, v.z, ysq);
                            ysq = fmaf(v.w, v.w, ysq);
                            sts4_u32((rpre ^ (uint32_t)(cc << 4)) + (uint32_t)(kb * OT_RB), v);
                        }
                    }
                }
                const float eps2 = a.eps * a.eps;
                int n = 0, status = 0;
                bool act = valid && !(ysq <= eps2 || ysq == 0.0f);
                float rsq = ysq;
                const float ynorm = sqrtf(ysq);
                // smallest decision margin relative to ||y|| (1: none close)
                float gmin = (a.eps > 0.f && ynorm > 0.f) ? fminf(1.0f, fabsf(ynorm - a.eps) / ynorm) : 1.0f;
                float L[CAP * (CAP + 1) / 2], invd[CAP], x[CAP], z[CAP];
                int ids[CAP];
#pragma unroll
                for (int t = 0; t < CAP; ++t) { ids[t] = -1; x[t] = 0.f; z[t] = 0.f; invd[t] = 0.f; }
#pragma unroll
                for (int t = 0; t < CAP * (CAP + 1) / 2; ++t) L[t] = 0.f;
                auto in_support = [&](int j) {
                    bool s = false;
#pragma unroll
                    for (int t = 0; t < CAP; ++t) s |= (ids[t] == j);
                    return s;
                };

                int cont = publish(act);
                while (cont) {
                    mbar_wait_sleep(smem_u32(&bars[B_FULL + g]), fph & 1u);
                    ++fph;
                    tmem_fence_after();
                    // ---------------- scan: ONE pass over the TMEM row. Block maxima
                    // (32 columns each); the block holding the running maximum is
                    // copied to the lane's shared-memory slot, so the candidates of
                    // the maximum's block come from the slot (every lane at once);
                    // only other blocks within the window (a near tie in another
                    // block) are re-read from TMEM, for the lanes that need them.
                    const float rn = sqrtf(rsq);
                    float thr = __int_as_float(0x7f800000);   // +inf: no candidates
                    float win = 0.f;
                    int nc = 0;
                    int cand[OT_CMAX];   // the OT_CMAX smallest candidate indices, ascending
#pragma unroll
                    for (int s = 0; s < OT_CMAX; ++s) cand[s] = 0x7fffffff;
                    // candidate j (not in the support): sorted insert, the largest index drops out
                    auto add = [&](int j) {
                        if (j < K && !in_support(j)) {
                            int x = j;
#pragma unroll
                            for (int s = 0; s < OT_CMAX; ++s) {
                                const int lo = min(cand[s], x);
                                x = max(cand[s], x);
                                cand[s] = lo;
                            }
                            ++nc;
                        }
                    };
                    auto extract = [&](const float (&v)[32], int j0) {
                        unsigned msk = 0u;
#pragma unroll
                        for (int t = 0; t < 32; ++t)
                            if (fabsf(v[t]) >= thr) msk |= 1u << t;
                        while (msk) {
                            const int j = j0 + __ffs(msk) - 1;
                            msk &= msk - 1u;
                            add(j);
                        }
                    };
                    if (__any_sync(SDB_FULL, act)) {
                        float bm[16];
                        float cmax = -1.f;
                        int sb = 0;
                        auto keep = [&](const uint32_t (&v)[32], int blk) {
                            float m0 = 0.f, m1 = 0.f;
#pragma unroll
                            for (int t = 0; t < 32; t += 2) {
                                m0 = fmaxf(m0, fabsf(__uint_as_float(v[t])));
                                m1 = fmaxf(m1, fabsf(__uint_as_float(v[t + 1])));
                            }
                            const float b = fmaxf(m0, m1);
                            bm[blk] = b;
                            if (b > cmax) {
                                cmax = b;
                                sb = blk;
#pragma unroll
                                for (int cc = 0; cc < 8; ++cc)
                                    sts4u_u32(slot + (uint32_t)(cc * OT_M * 16), v[4 * cc], v[4 * cc + 1], v[4 * cc + 2],
                                              v[4 * cc + 3]);
                            }
                        };
                        // the TMEM load of the next block is in flight while this one
                        // is reduced (two register buffers)
                        constexpr int NB = NCH * 8;
                        const int nblk = ((K + 63) >> 6) << 1;   // blocks holding atoms (in pairs)
                        auto tcol = [&](int blk) -> uint32_t {
                            return trow + (uint32_t)((NCH == 2 ? (blk >> 3) : (g & 1)) * OT_N + (blk & 7) * 32);
                        };
#pragma unroll
                        for (int blk = 0; blk < 16; ++blk) bm[blk] = 0.f;
                        {
                            uint32_t va[32], vb[32];
                            tmem_ld32(va, tcol(0));
#pragma unroll
                            for (int blk = 0; blk < NB; blk += 2) {
                                if (blk < nblk) {
                                    tmem_wait_ld();
                                    tmem_ld32(vb, tcol(blk + 1));
                                    keep(va, blk);
                                    tmem_wait_ld();
                                    if (blk + 2 < NB && blk + 2 < nblk) tmem_ld32(va, tcol(blk + 2));
                                    keep(vb, blk + 1);
                                }
                            }
                        }
                        win = OT_WIN * rn + 1e-6f * ynorm;
                        // a maximum below the window itself (a residual at rounding
                        // level, e.g. a signal that is one of the dictionary's atoms):
                        // EVERY atom is within the window, and the OT_CMAX lowest
                        // candidates -- all that is kept -- are in block 0, so only
                        // that block is walked instead of all K columns
                        if (act) thr = cmax - win;
                        const bool allin = act && thr < 0.f;
                        if (act && (!allin || sb == 0)) {
                            float v[32];
#pragma unroll
                            for (int cc = 0; cc < 8; ++cc) {
                                const float4 f = lds4_u32(slot + (uint32_t)(cc * OT_M * 16));
                                v[4 * cc] = f.x;
                                v[4 * cc + 1] = f.y;
                                v[4 * cc + 2] = f.z;
                                v[4 * cc + 3] = f.w;
                            }
                            extract(v, sb * 32);
                        }
                        // other blocks within the window (the lane's own need mask; the
                        // warp re-reads the union of them)
                        unsigned need = 0u;
#pragma unroll
                        for (int blk = 0; blk < 16; ++blk)
                            if ((blk >> 3) < NCH && blk * 32 < K && bm[blk] >= thr && blk != sb) need |= 1u << blk;
                        if (allin) need &= 1u;
                        unsigned wneed = __reduce_or_sync(SDB_FULL, need);
#pragma unroll 1
                        while (wneed) {
                            const int blk = __ffs(wneed) - 1;
                            wneed &= wneed - 1u;
                            uint32_t u[32];
                            const uint32_t col = (uint32_t)((NCH == 2 ? (blk >> 3) : (g & 1)) * OT_N + (blk & 7) * 32);
                            tmem_ld32(u, trow + col);
                            tmem_wait_ld();
                            if ((need >> blk) & 1u) {
                                float v[32];
#pragma unroll
                                for (int t = 0; t < 32; ++t) v[t] = __uint_as_float(u[t]);
                                extract(v, blk * 32);
                            }
                        }
                    }
                    // the chunk buffers go back to the MMA issuer
                    tmem_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        for (int c = 0; c < NCH; ++c) mbar_arrive(smem_u32(&bars[B_EMPTY + (NCH == 2 ? c : (g & 1))]));
                    }
                    if (act) {
                        // ---------------- exact selection among the candidates
                        float best = -1.f, second = -1.f, eb = 0.f;
                        int bj = -1;
                        auto consider = [&](int j) {
                            const float d = dot(j);
                            const float ad = fabsf(d);
                            if (ad > best || (ad == best && j < bj)) {
                                second = best;
                                best = ad;
                                eb = d;
                                bj = j;
                            } else if (ad > second) {
                                second = ad;
                            }
                        };
                        // a residual at rounding level (every |corr| below the margin
                        // floor 1e-6 ||y||): the choice among the many in-window atoms is
                        // noise for the reference as well (such steps are excluded from
                        // the decision margin and their coefficients refit to ~0 in FP64),
                        // so the listed candidates are refined instead of all K atoms
                        const bool noise = (thr + win) < 1e-6f * ynorm;
                        if (nc >= 1 && (nc <= OT_CMAX || noise)) {
                            // one inlined refinement: the list is consumed from the front
                            const int ncl = min(nc, OT_CMAX);
#pragma unroll 1
                            for (int s = 0; s < ncl; ++s) {
                                consider(cand[0]);
#pragma unroll
                                for (int q = 0; q + 1 < OT_CMAX; ++q) cand[q] = cand[q + 1];
                            }
                            // every non-candidate atom has |d.r| < thr + win/2
                            second = fmaxf(second, thr + 0.5f * win);
                        } else {
                            for (int j = 0; j < K; ++j)
                                if (!in_support(j)) consider(j);
                        }
                        if (noise && nc > OT_CMAX) {
                            // not every in-window atom was refined: a non-negligible
                            // best (borderline) cannot be certified here -> FP64 re-run
                            if (best >= 1e-6f * ynorm) gmin = 0.f;
                        } else if (best >= 1e-6f * ynorm) {
                            gmin = fminf(gmin, fmaxf(0.f, best - second) / ynorm);
                        }
                        if (bj < 0 || best * best <= 1e-26f * rsq) {   // cmax <= 1e-13 ||r|| (_kernels.py:97)
                            status = 3;
                            act = false;
                        } else {
                            // ---------------- Cholesky append (_kernels.py:109-127) and the
                            // solve (_kernels.py:129-139), specialised on the support size
                            // n0 (every active lane of the warp is at the same step, so the
                            // switch is uniform): static triangular indices, no padding terms
                            float dx[CAP];
#pragma unroll
                            for (int t = 0; t < CAP; ++t) dx[t] = 0.f;
                            auto append = [&](auto nc) -> bool {
                                constexpr int n0 = decltype(nc)::value;
                                const float* __restrict__ Gb = Gp + (int64_t)bj * K;
                                const float gbb = __ldg(Gb + bj);
                                float gb[n0 + 1], w[n0 + 1];
#pragma unroll
                                for (int t = 0; t < n0; ++t) gb[t] = __ldg(Gb + ids[t]);
                                float c0b = eb;   // d_b.y = d_b.r + G[b,S] x
#pragma unroll
                                for (int t = 0; t < n0; ++t) c0b = fmaf(gb[t], x[t], c0b);
                                float dsq = gbb;
#pragma unroll
                                for (int t = 0; t < n0; ++t) {
                                    float acc = gb[t];
#pragma unroll
                                    for (int u = 0; u < t; ++u) acc = fmaf(-L[t * (t + 1) / 2 + u], w[u], acc);
                                    w[t] = acc * invd[t];
                                    dsq = fmaf(-w[t], w[t], dsq);
                                }
                                if (dsq <= a.guard) return false;   // numerically singular support Gram
                                const float inv = rsqrtf(dsq);
                                float zn = c0b;
#pragma unroll
                                for (int t = 0; t < n0; ++t) zn = fmaf(-w[t], z[t], zn);
                                zn *= inv;
#pragma unroll
                                for (int t = 0; t < n0; ++t) L[n0 * (n0 + 1) / 2 + t] = w[t];
                                L[n0 * (n0 + 1) / 2 + n0] = dsq * inv;
                                invd[n0] = inv;
                                ids[n0] = bj;
                                z[n0] = zn;
                                // back substitution L^T x = z
                                float xn[n0 + 1];
#pragma unroll
                                for (int t = n0; t >= 0; --t) {
                                    float acc = z[t];
#pragma unroll
                                    for (int u = t + 1; u <= n0; ++u) acc = fmaf(-L[u * (u + 1) / 2 + t], xn[u], acc);
                                    xn[t] = acc * invd[t];
                                }
#pragma unroll
                                for (int t = 0; t <= n0; ++t) {
                                    dx[t] = xn[t] - x[t];
                                    x[t] = xn[t];
                                }
                                return true;
                            };
                            bool ok = false;
                            switch (n) {
#define SDB_OT_CASE(I) \
    case I:            \
        if constexpr (I < CAP) ok = append(std::integral_constant<int, I>{}); \
        break;
                                SDB_OT_CASE(0) SDB_OT_CASE(1) SDB_OT_CASE(2) SDB_OT_CASE(3)
                                SDB_OT_CASE(4) SDB_OT_CASE(5) SDB_OT_CASE(6) SDB_OT_CASE(7)
#undef SDB_OT_CASE
                                default: break;
                            }
                            if (!ok) {
                                status = 2;
                                act = false;
                            } else {
                                ++n;
                                const bool need_r = n < a.cap || a.rnorm != nullptr || a.eps > 0.f;
                                if (need_r) {
                                    // r -= D_S dx in place (the next MMA's A operand), one
                                    // k-block (32 floats in registers) at a time. Every active
                                    // lane of the warp is at the same step, so the branches on
                                    // t < n are uniform
                                    float r0 = 0.f, r1 = 0.f;
#pragma unroll
                                    for (int kb = 0; kb < NKB; ++kb) {
                                        float4 v[8];
#pragma unroll
                                        for (int cc = 0; cc < 8; ++cc)
                                            v[cc] = lds4_u32((rpre ^ (uint32_t)(cc << 4)) + (uint32_t)(kb * OT_RB));
#pragma unroll
                                        for (int t = 0; t < CAP; ++t) {
                                            if (t < n) {
                                                const uint32_t dp = dpre(ids[t]);
                                                const float c = -dx[t];
#pragma unroll
                                                for (int cc = 0; cc < 8; ++cc) {
                                                    const float4 d = lds4_u32((dp ^ (uint32_t)(cc << 4)) +
                                                                              (uint32_t)(kb * KPAD * 128));
                                                    v[cc].x = fmaf(c, d.x, v[cc].x);
                                                    v[cc].y = fmaf(c, d.y, v[cc].y);
                                                    v[cc].z = fmaf(c, d.z, v[cc].z);
                                                    v[cc].w = fmaf(c, d.w, v[cc].w);
                                                }
                                            }
                                        }
#pragma unroll
                                        for (int cc = 0; cc < 8; ++cc) {
                                            sts4_u32((rpre ^ (uint32_t)(cc << 4)) + (uint32_t)(kb * OT_RB), v[cc]);
                                            r0 = fmaf(v[cc].x, v[cc].x, r0);
                                            r1 = fmaf(v[cc].y, v[cc].y, r1);
                                            r0 = fmaf(v[cc].z, v[cc].z, r0);
                                            r1 = fmaf(v[cc].w, v[cc].w, r1);
                                        }
                                    }
                                    rsq = r0 + r1;
                                }
                                if (a.eps > 0.f) gmin = fminf(gmin, fabsf(__fsqrt_rn(rsq) - a.eps) / ynorm);
                                if (n >= a.cap) act = false;
                                else if (__fsqrt_rn(rsq) <= a.eps) act = false;   // _kernels.py:153
                            }
                        }
                    }
                    cont = publish(act);
                }
                // the MMA issuer's acknowledgement of the tile end
                mbar_wait_sleep(smem_u32(&bars[B_FULL + g]), fph & 1u);
                ++fph;
                // ---- codes in selection order (entries >= n zeroed like the reference)
                if (valid) {
                    int32_t* ci = a.idx + i * a.cap;
                    float* cv = a.val + i * a.cap;
#pragma unroll
                    for (int t = 0; t < CAP; ++t) {
                        if (t < a.cap) {
                            ci[t] = (t < n) ? ids[t] : 0;
                            cv[t] = (t < n) ? x[t] : 0.f;
                        }
                    }
                    a.counts[i] = n;
                    a.status[i] = (int8_t)status;
                    if (a.rnorm) a.rnorm[i] = __fsqrt_rn(rsq);
                    if (a.gap) a.gap[i] = gmin;
                }
            }
            if (rd.last) {
                // this group no longer reads the shard's dictionary
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars[B_DFREE]));
            }
        }
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * OT_N));
}

// D (P x K x m fp32, atom-major) -> P x kpad x m_pad, zero padded
__global__ void k_pad_dict(int64_t P, int K, int m, int kpad, int m_pad, const float* __restrict__ D,
                           float* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tot = P * kpad * m_pad;
    if (e >= tot) return;
    const int c = (int)(e % m_pad);
    const int64_t rr = e / m_pad;
    const int j = (int)(rr % kpad);
    const int64_t p = rr / kpad;
    out[e] = (j < K && c < m) ? D[(p * K + j) * m + c] : 0.0f;
}

__global__ void k_omp_tc_tiles(const int64_t* __restrict__ off, int P, int64_t* __restrict__ ts) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t t = 0;
        for (int p = 0; p < P; ++p) {
            ts[p] = t;
            t += (off[p + 1] - off[p] + OT_M - 1) / OT_M;
        }
        ts[P] = t;
    }
}

inline int64_t al256(int64_t b) { return (b + 255) & ~int64_t(255); }

}  // namespace

bool omp_tc_supported(int64_t m, int64_t K, int64_t cap) {
    return m >= 1 && m <= 64 && K >= 1 && K <= 512 && cap >= 1 && cap <= 8;
}

int64_t omp_tc_ws_bytes(int64_t P, int64_t m, int64_t K) {
    const int64_t m_pad = (m + 31) / 32 * 32, kpad = (K + OT_N - 1) / OT_N * OT_N;
    return al256(P * kpad * m_pad * 4) + al256(8 * (P + 1));
}

int omp_tc_f32(int64_t N, int m, int K, int P, const int64_t* off, const float* Y, int64_t ldy, const float* D,
               const float* G, int cap, float eps, float guard, int32_t* idx, float* val, int32_t* counts,
               int8_t* status, float* rnorm, float* gap, void* ws, int64_t ws_bytes, cudaStream_t st) {
    if (!omp_tc_supported(m, K, cap)) return (int)cudaErrorNotSupported;
    if (N <= 0) return 0;
    if (ws == nullptr || ws_bytes < omp_tc_ws_bytes(P, m, K)) return (int)cudaErrorInvalidValue;
    const int m_pad = (m + 31) / 32 * 32;
    const int nch = (K + OT_N - 1) / OT_N;
    const int kpad = nch * OT_N;
    float* Dp = (float*)ws;
    int64_t* ts = (int64_t*)((unsigned char*)ws + al256((int64_t)P * kpad * m_pad * 4));
    const int64_t tot = (int64_t)P * kpad * m_pad;
    k_pad_dict<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(P, K, m, kpad, m_pad, D, Dp);
    k_omp_tc_tiles<<<1, 32, 0, st>>>(off, P, ts);
    CUtensorMap mD;
    if (!tc_map_f32(&mD, Dp, m_pad, (int64_t)P * kpad, m_pad, OT_N)) return (int)cudaErrorNotSupported;
    OtArgs a{};
    a.N = N; a.m = m; a.K = K; a.P = P; a.cap = cap; a.nkb = m_pad / 32; a.nch = nch; a.kpad = kpad;
    a.off = off; a.ts = ts; a.Y = Y; a.ldy = ldy; a.G = G; a.eps = eps; a.guard = guard;
    a.idx = idx; a.val = val; a.counts = counts; a.status = status; a.rnorm = rnorm; a.gap = gap;
    // three signal groups are possible when K > 256 (the groups share both
    // TMEM chunk buffers anyway) and the residual tiles fit next to the
    // dictionary; measured no faster than two at C4 (the tile-steps serialise
    // on the TMEM accumulator, and 128 registers spill), so opt-in only
    const int smem3 = 1024 + a.nkb * kpad * 128 + 3 * (a.nkb * OT_RB + OT_M * 128) + 256;
    static const bool want3 = getenv("SDB_OMP_TC_3GRP") != nullptr;
    const bool three = want3 && nch == 2 && smem3 <= 232448;
    const int ng = three ? 3 : 2;
    const int smem = 1024 + a.nkb * kpad * 128 + ng * (a.nkb * OT_RB + OT_M * 128) + 256;
    int dev = 0;
    cudaGetDevice(&dev);
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    using Fn = void (*)(const CUtensorMap, const OtArgs);
    Fn fn = nullptr;
#define SDB_OT_PICK(C, G, B, H) \
    if ((cap <= 4 ? 4 : 8) == C && ng == G && a.nkb == B && nch == H) fn = k_omp_tc<C, G, B, H>;
    SDB_OT_PICK(4, 2, 1, 1) SDB_OT_PICK(4, 2, 2, 1) SDB_OT_PICK(4, 2, 1, 2) SDB_OT_PICK(4, 2, 2, 2)
    SDB_OT_PICK(8, 2, 1, 1) SDB_OT_PICK(8, 2, 2, 1) SDB_OT_PICK(8, 2, 1, 2) SDB_OT_PICK(8, 2, 2, 2)
    SDB_OT_PICK(4, 3, 1, 2) SDB_OT_PICK(4, 3, 2, 2) SDB_OT_PICK(8, 3, 1, 2) SDB_OT_PICK(8, 3, 2, 2)
#undef SDB_OT_PICK
    if (fn == nullptr) return (int)cudaErrorNotSupported;
    cudaError_t e = set_max_smem((const void*)fn, smem);
    if (e != cudaSuccess) return (int)e;
    const int64_t max_tiles = (N + OT_M - 1) / OT_M + P;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(n_sm, max_tiles));
    // chunk length of the round-robin tile assignment. Gram matrices that fit
    // in L2 together: one contiguous range per CTA (fewest dictionary loads).
    // Otherwise a few rounds per chunk, so the grid stays on a handful of
    // shards: the longest of 1..4 rounds within 2% of the best balance
    static const int clen_env = getenv("SDB_OMP_TC_CLEN") ? atoi(getenv("SDB_OMP_TC_CLEN")) : 0;
    const int64_t per = (max_tiles + grid - 1) / grid;
    int64_t clen = per;
    if ((int64_t)P * K * K * 4 > (int64_t)16 << 20) {
        auto worst = [&](int64_t c) { return ((max_tiles + c - 1) / c + grid - 1) / grid * c; };
        int64_t best = INT64_MAX;
        for (int r = 1; r <= 4; ++r) best = std::min(best, worst((int64_t)r * ng));
        for (int r = 4; r >= 1; --r) {
            clen = (int64_t)r * ng;
            if (worst(clen) * 100 <= best * 102) break;
        }
    }
    a.clen = clen_env > 0 ? clen_env : (int)std::min<int64_t>(clen, 1 << 30);
    fn<<<grid, (2 + 4 * ng) * 32, smem, st>>>(mD, a);
    return (int)cudaGetLastError();
}

}  // namespace sdb
