// Correlation GEMM on the 5th-gen tensor cores (sm_100a):
//   alpha0[i, j] = <y_i, d_j>   for every signal i, atom j of i's shard
// i.e. the c0 = D^T y loop of omp_single (_kernels.py:54-59) for a whole
// batch, in 3xTF32 split precision (FP32-level accuracy on TF32 units):
//   y = y_hi + y_lo, d = d_hi + d_lo (hi = tf32 round-to-nearest)
//   alpha0 ~= y_hi.d_hi + y_hi.d_lo + y_lo.d_hi   (FP32 accumulation in TMEM)
//
// Work item = (128-signal tile, 256-atom chunk, shard): TMA
// (cp.async.bulk.tensor, 128B swizzle) streams 32-wide k-blocks of Y (fp32)
// and of the pre-split D_hi / D_lo into a 2-stage smem ring guarded by
// mbarriers; the Y k-block is split into hi/lo in place (element-wise, so the
// swizzled layout is preserved); one elected thread issues 4 k-steps x 3
// tcgen05.mma.kind::tf32 (M=128, N=256, K=8) into a TMEM accumulator; the
// epilogue drains TMEM through swizzled smem into TMA stores.
#include <cuda.h>

#include <cstdint>
#include <algorithm>
#include <mutex>

#include "sdb_common.cuh"
#include "sdb_internal.h"
#include "sdb_tc.cuh"

namespace sdb {

namespace {

constexpr int TM = 128;      // signals per tile (UMMA M)
constexpr int TN = 256;      // atoms per chunk (UMMA N)
constexpr int KB = 32;       // fp32 elements per 128-byte swizzle row
constexpr int A_BYTES = TM * KB * 4;   // 16 KB
constexpr int B_BYTES = TN * KB * 4;   // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B_hi, B_lo

}  // namespace

// ----------------------------------------------------------------------------
// Persistent, warp-specialised version (the one used): one CTA per SM owns a
// contiguous range of work items ordered (shard, 256-atom chunk, 128-signal
// tile); roles:
//   warp 0      TMA producer (one elected thread)
//   warp 1      MMA issuer (one thread): 4 k-steps x 3 MMAs per k-block
//   warps 2-5   epilogue: TMEM -> registers -> global (thread = signal row)
//   warps 6-9   3xTF32 split of the Y k-block (hi in place, lo beside it)
// RES (m <= 64): D_hi/D_lo of the current (shard, chunk) stay resident in
// smem and are reloaded only when the segment changes; the 2-stage ring then
// carries Y only. !RES: D k-blocks stream with Y through the ring.
// The accumulator is double-buffered in TMEM (2 x 256 columns), so the
// epilogue of item i overlaps the loads and MMAs of item i+1.
// mbarriers: full[s] (TMA), split[s] (4 warps), empty[s] (MMA commit),
//            tfull[b] (MMA commit), tempty[b] (4 epilogue warps),
//            bfull (resident D landed), bfree (MMA done with resident D).
// ----------------------------------------------------------------------------
constexpr int NWARP2 = 14;  // warps 10-13: second epilogue half (CODE only)
constexpr int RES_KB = 2;                           // resident D: up to 2 k-blocks (m <= 64)
constexpr int RES_A_STAGE = 2 * A_BYTES;             // Y hi + lo
constexpr int RES_B_BYTES = RES_KB * 2 * B_BYTES;    // D hi + lo, 2 k-blocks
// + TMA store staging (1024-aligned for the 128-byte swizzle)
constexpr int SMEM2_BYTES = 2 * STAGE_BYTES + 1024 + 1024 + 4 * 2 * 32 * 32 * 4;
// shared memory per variant (CODE needs no TMA-store staging; a third Y stage
// fits there for RES but measured no faster: the MMA is tensor-pipe bound)
template <bool RES, bool CODE>
struct Cfg {
    static constexpr int NST = 2;
    static constexpr int DATA = RES ? NST * RES_A_STAGE + RES_KB * 2 * B_BYTES : 2 * STAGE_BYTES;
    static constexpr int XCHG = 4 * 400 + 4 * 1024;            // CODE: pair exchange + per-warp G diagonal
    static constexpr int SMEM = 1024 + DATA + (CODE ? 256 + XCHG : 1024 + 4 * 2 * 32 * 32 * 4);
};
static_assert(Cfg<true, true>::SMEM <= 232448, "smem");


struct Item {
    int p, chunk;
    int64_t tile, seg;  // seg: (p, chunk) segment id
};

__device__ __forceinline__ Item item_of(int64_t it, const int64_t* __restrict__ tile_start, int P,
                                        int nchunk) {
    // items of shard p: nchunk * ntiles_p, ordered (chunk, tile)
    int lo = 0, hi = P - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] * nchunk <= it) lo = mid; else hi = mid - 1;
    }
    Item r;
    r.p = lo;
    const int64_t nt = tile_start[lo + 1] - tile_start[lo];
    const int64_t local = it - tile_start[lo] * nchunk;
    r.chunk = (int)(local / nt);
    r.tile = local - (int64_t)r.chunk * nt;
    r.seg = (int64_t)lo * nchunk + r.chunk;
    return r;
}

// A role's walk over its consecutive items: one search for the first item, then
// (tile, chunk, shard) advance in place (the search is ~5 dependent loads and a
// 64-bit division per item otherwise)
struct ItemWalk {
    Item I;
    int64_t nt;   // tiles of the current shard
    __device__ __forceinline__ ItemWalk(int64_t it, int64_t it_end, const int64_t* __restrict__ tile_start, int P,
                                        int nchunk) {
        if (it < it_end) {
            I = item_of(it, tile_start, P, nchunk);
            nt = tile_start[I.p + 1] - tile_start[I.p];
        } else {
            I.p = 0; I.chunk = 0; I.tile = 0; I.seg = 0;
            nt = 1;
        }
    }
    // the next item starts another (shard, chunk) segment
    __device__ __forceinline__ bool seg_ends() const { return I.tile + 1 >= nt; }
    __device__ __forceinline__ void next(const int64_t* __restrict__ tile_start, int P, int nchunk) {
        if (++I.tile < nt) return;
        I.tile = 0;
        if (++I.chunk >= nchunk) {
            I.chunk = 0;
            do {   // empty shards own no items
                ++I.p;
                nt = I.p < P ? tile_start[I.p + 1] - tile_start[I.p] : 1;
            } while (I.p < P && nt == 0);
        }
        I.seg = (int64_t)I.p * nchunk + I.chunk;
    }
};

// CODE: the epilogue also runs the first greedy step of the error-bounded
// FP32 OMP (k_omp_fast, sdb_omp.cu) on each signal's TMEM row, with the same
// arithmetic: argmax |alpha0| (lowest index among equal maxima), stall and
// singular tests, x = c0[b] / G[b,b], ||r||^2 = ||y||^2 - c0[b]^2 / G[b,b].
// A signal that this settles (no atom, one atom, or a stop status) gets its
// code row, count and status written here and its alpha0 row is never
// stored; every other signal (a second atom is needed, or ||r|| is within
// the band where the explicit residual decides) has its alpha0 row stored
// and status -1, and k_omp_fast<DEFER> codes it from scratch. Needs K <= 256
// (the whole row in one accumulator).
struct Step1 {
    const float* ysq;     // N: ||y||^2 (sdb_signal_sq)
    const float* G;       // P x K x K
    float eps2, guard;
    int cap;
    int32_t* idx;         // N x cap
    float* val;           // N x cap
    int32_t* counts;
    int8_t* status;
    int* n_deferred;      // zeroed by k_tile_layout
    float* gap;           // optional: settled signals' smallest decision margin / ||y|| (certification)
};

// argmax |x| over one 32-column block of a row: a pairwise tree on the raw
// values compared by magnitude (the left, lower-index operand wins ties, so
// the result is the lowest index attaining the maximum, as the reference's
// ascending scan gives). Columns past K enter as 0, which is never selected
// (selection needs |x| > the running maximum >= 0). alpha0 is finite here:
// rows whose ||y||^2 is not finite are deferred before this is consulted.
// SECOND: also the block's runner-up magnitude (certification margin). Every
// element but the winner loses exactly one comparison of the tree and the
// second largest loses only to the winner, so the runner-up is the largest
// loser -- one min and one max per comparison instead of a second pass over
// the block (a second element equal to the maximum is a loser too).
template <bool FULL, bool SECOND>
__device__ __forceinline__ void block_argmax(const uint32_t (&v)[32], int c, int K, float& bx, uint32_t& bk,
                                             float& bs) {
    float a[32];
    uint32_t k[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        a[t] = (FULL || c + t < K) ? __uint_as_float(v[t]) : 0.0f;
        k[t] = (uint32_t)t;
    }
    float l0 = 0.0f, l1 = 0.0f;
#pragma unroll
    for (int w = 1; w < 32; w <<= 1)
#pragma unroll
        for (int t = 0; t < 32; t += 2 * w) {
            const bool r = fabsf(a[t + w]) > fabsf(a[t]);
            if (SECOND) {
                const float lo = fminf(fabsf(a[t + w]), fabsf(a[t]));
                if ((t / (2 * w)) & 1) l1 = fmaxf(l1, lo); else l0 = fmaxf(l0, lo);
            }
            a[t] = r ? a[t + w] : a[t];
            k[t] = r ? k[t + w] : k[t];
        }
    bx = a[0];
    bk = k[0] + (uint32_t)c;
    bs = fmaxf(l0, l1);
}

__device__ __forceinline__ void pair_sync(int quad) {
    // the two epilogue warps of one TMEM lane quadrant (named barrier 1 + quad)
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
}

// Step-1 epilogue for 32 signal rows (thread = row_base + lane) of a K <= 256
// accumulator, split over the two warps of the lane quadrant: warp half h
// scans columns [c_lo, c_hi); the halves meet in shared memory (xv/xk: the
// upper half's per-row signed maximum and its column, *xm: the deferred-row
// mask). diag: the lower warp's smem copy of the shard's G diagonal; ysq:
// ||y||^2 of the lower warp's rows, fetched before the accumulator wait.
__device__ __forceinline__ void code_step1(const Step1& s1, uint32_t trow, int64_t row_base, int nrows,
                                           int p, int K, int half, int c_lo, int c_hi,
                                           float* xv, uint32_t* xk, unsigned* xm, const float* diag,
                                           float ysq, int quad,
                                           float* __restrict__ alpha, int64_t lda, int lane) {
    const int64_t i = row_base + lane;
    const bool valid = lane < nrows;
    // ---- argmax |alpha0| over this warp's columns (and, for certification,
    // the runner-up magnitude)
    float cur = 0.0f, cx = 0.0f;      // running max |alpha0|, its signed value
    float sec = 0.0f;                 // running second-largest |alpha0| (s1.gap only)
    uint32_t key = 0xffffffffu;
    uint32_t va[32], vb[32];
    const bool margin = s1.gap != nullptr;
    auto scan = [&](const uint32_t (&v)[32], int c) {
        float bx, bs;
        uint32_t bk;
        if (margin) {   // warp-uniform
            if (c + 32 <= K) block_argmax<true, true>(v, c, K, bx, bk, bs);
            else block_argmax<false, true>(v, c, K, bx, bk, bs);
            sec = fmaxf(fmaxf(sec, bs), fminf(cur, fabsf(bx)));
        } else {
            if (c + 32 <= K) block_argmax<true, false>(v, c, K, bx, bk, bs);
            else block_argmax<false, false>(v, c, K, bx, bk, bs);
        }
        if (fabsf(bx) > cur) { cur = fabsf(bx); cx = bx; key = bk; }
    };
    // 32-column blocks, the next block's TMEM load in flight during each scan
    if (c_lo < c_hi) {
        tmem_ld32(va, trow + (uint32_t)c_lo);
        tmem_wait_ld();
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 64) {
            if (c + 32 < c_hi) tmem_ld32(vb, trow + (uint32_t)(c + 32));
            scan(va, c);
            tmem_wait_ld();
            if (c + 32 >= c_hi) break;
            if (c + 64 < c_hi) tmem_ld32(va, trow + (uint32_t)(c + 64));
            scan(vb, c + 32);
            tmem_wait_ld();
        }
    }
    // ---- combine the halves (the lower half's columns win ties)
    float* xs = xv + 68;              // upper half's runner-up (certification)
    if (half == 1) { xv[lane] = cx; xk[lane] = key; if (margin) xs[lane] = sec; }
    pair_sync(quad);
    bool defer = false;
    unsigned dmask;
    if (half == 0) {
        const float cu = xv[lane];
        const uint32_t ku = xk[lane];
        if (margin) sec = fmaxf(fmaxf(sec, xs[lane]), fminf(cur, fabsf(cu)));
        if (fabsf(cu) > cur) { cur = fabsf(cu); cx = cu; key = ku; }
        const float ynrm = sqrtf(ysq);
        float gm = 1.0f;
        if (margin && ynrm > 0.0f) {
            const float eps = sqrtf(s1.eps2);
            if (eps > 0.0f) gm = fminf(gm, fabsf(ynrm - eps) / ynrm);
            if (cur >= 1e-6f * ynrm) gm = fminf(gm, (cur - sec) / ynrm);
        }
        // ---- the first greedy step (k_omp_fast, step 0); the deferral mask
        // is published before any store, so the upper warp is released early
        int n = 0, status = 0, best = 0;
        float x0 = 0.0f;
        if (valid) {
            if (ysq <= s1.eps2 || ysq == 0.0f) {
                // ||y|| <= eps: no atom
            } else if (!(ysq <= 3.0e38f)) {
                defer = true;                     // ||y||^2 not finite: alpha0 may be too; k_omp_fast decides
            } else if (cur * cur <= 1e-26f * ysq) {
                status = 3;                       // cmax <= 1e-13 ||r|| (also: no candidate)
            } else {
                best = (int)key;
                const float cb = cx;
                const float dsq = diag[best];
                if (dsq <= s1.guard) {
                    status = 2;
                    best = 0;
                } else {
                    const float inv = rsqrtf(dsq);
                    const float tn = cb * inv;
                    x0 = tn * inv;
                    n = 1;
                    const float rsq = fmaxf(fmaf(-tn, tn, ysq), 0.0f);
                    if (s1.cap > 1 && (fabsf(rsq - s1.eps2) <= 1e-4f * ysq || rsq > s1.eps2)) defer = true;
                    if (margin) gm = fminf(gm, fabsf(sqrtf(rsq) - sqrtf(s1.eps2)) / ynrm);
                }
            }
        }
        dmask = __ballot_sync(SDB_FULL, defer);
        if (lane == 0) *xm = dmask;
        pair_sync(quad);
        if (lane == 0 && dmask) atomicAdd(s1.n_deferred, __popc(dmask));   // result unused: a fire-and-forget RED
        if (valid) {
            if (!defer) {
                int32_t* ci = s1.idx + i * s1.cap;
                float* cv = s1.val + i * s1.cap;
                if ((s1.cap & 3) == 0) {
                    int4* ci4 = reinterpret_cast<int4*>(ci);
                    float4* cv4 = reinterpret_cast<float4*>(cv);
                    ci4[0] = make_int4(best, 0, 0, 0);
                    cv4[0] = make_float4(x0, 0.0f, 0.0f, 0.0f);
                    for (int t = 1; t < (s1.cap >> 2); ++t) {
                        ci4[t] = make_int4(0, 0, 0, 0);
                        cv4[t] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    }
                } else {
                    for (int t = 0; t < s1.cap; ++t) {
                        ci[t] = (t < n) ? best : 0;
                        cv[t] = (t < n) ? x0 : 0.0f;
                    }
                }
                s1.counts[i] = n;
                if (margin) s1.gap[i] = gm;
            }
            s1.status[i] = defer ? (int8_t)-1 : (int8_t)status;
        }
    } else {
        pair_sync(quad);
    }
    if (half == 1) {
        dmask = *xm;
        defer = (dmask >> lane) & 1u;
    }
    // ---- deferred rows: this warp's columns of the alpha0 row, each thread
    // its own (8 x 16-byte stores fill one 128-byte line per 32 columns)
    if (dmask == 0u || c_lo >= c_hi) return;
    float* out = alpha + i * lda;
    auto put = [&](const uint32_t (&v)[32], int c) {
        if (!defer) return;
        if (c + 32 <= K) {
            float4* o4 = reinterpret_cast<float4*>(out + c);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                o4[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                    __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        } else {
#pragma unroll
            for (int q = 0; q < 32; ++q)
                if (c + q < K) out[c + q] = __uint_as_float(v[q]);
        }
    };
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += 64) {
        if (c + 32 < c_hi) {
            tmem_ld64(va, vb, trow + (uint32_t)c);
            tmem_wait_ld();
            put(va, c);
            put(vb, c + 32);
        } else {
            tmem_ld32(va, trow + (uint32_t)c);
            tmem_wait_ld();
            put(va, c);
        }
    }
}

template <bool RES, bool CODE>
__global__ void __launch_bounds__(NWARP2 * 32, 1)
k_corr_tc2(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmDh,
           const __grid_constant__ CUtensorMap tmDl, const __grid_constant__ CUtensorMap tmA,
           const int64_t* __restrict__ off,
           const int64_t* __restrict__ tile_start, int P, int K, int nkb, int nchunk,
           float* __restrict__ alpha, int64_t lda, const Step1 s1) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr int NST = Cfg<RES, CODE>::NST;
    // layout: RES: [A stage 0 .. NST-1 | D resident] ; !RES: [stage 0 | stage 1]
    unsigned char* bar_base = base + Cfg<RES, CODE>::DATA;
    uint64_t* bars = (uint64_t*)bar_base;
    // full[s] = s, split[s] = NST + s, empty[s] = 2 NST + s, tfull[b] = 3 NST + b,
    // tempty[b] = 3 NST + 2 + b, bfull = 3 NST + 4, bfree = 3 NST + 5
    constexpr int B_SPLIT = NST, B_EMPTY = 2 * NST, B_TFULL = 3 * NST, B_TEMPTY = 3 * NST + 2;
    constexpr int B_BFULL = 3 * NST + 4, B_BFREE = 3 * NST + 5;
    uint32_t* tmem_slot = (uint32_t*)(bars + 3 * NST + 6);
    // epilogue staging for TMA stores: 4 warps x 2 buffers x 32x32 fp32,
    // 128-byte swizzled (row r's 16-byte chunk c at c ^ (r & 7)); CODE: the
    // pair exchange slots instead
    float* stg_base = reinterpret_cast<float*>(bar_base + (CODE ? 256 : 1024));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n_items = tile_start[P] * nchunk;
    const int64_t per = (n_items + gridDim.x - 1) / gridDim.x;
    const int64_t it0 = (int64_t)blockIdx.x * per, it1 = min(n_items, it0 + per);

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[B_SPLIT + s]), 4);
            mbar_init(smem_u32(&bars[B_EMPTY + s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bars[B_TFULL + b]), 1);
            mbar_init(smem_u32(&bars[B_TEMPTY + b]), CODE ? 8 : 4);
        }
        mbar_init(smem_u32(&bars[B_BFULL]), 1);
        mbar_init(smem_u32(&bars[B_BFREE]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "r"(2 * TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    // A (Y) k-block buffers of stage s; D k-block kb buffers (resident or staged)
    auto a_hi = [&](int s) -> unsigned char* { return RES ? base + s * RES_A_STAGE : base + s * STAGE_BYTES; };
    auto a_lo = [&](int s) -> unsigned char* { return a_hi(s) + A_BYTES; };
    auto b_hi = [&](int s, int kb) -> unsigned char* {
        return RES ? base + NST * RES_A_STAGE + kb * 2 * B_BYTES : base + s * STAGE_BYTES + 2 * A_BYTES;
    };
    auto b_lo = [&](int s, int kb) -> unsigned char* { return b_hi(s, kb) + B_BYTES; };

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int64_t q = 0, seg_prev = -1, nseg = 0;
            ItemWalk W(it0, it1, tile_start, P, nchunk);
            for (int64_t it = it0; it < it1; ++it, W.next(tile_start, P, nchunk)) {
                const Item I = W.I;
                const int64_t row0 = off[I.p] + I.tile * TM;
                const int64_t d_row0 = (int64_t)I.p * K + (int64_t)I.chunk * TN;
                if (RES && I.seg != seg_prev) {
                    if (nseg > 0) mbar_wait(smem_u32(&bars[B_BFREE]), (uint32_t)((nseg - 1) & 1));
                    const uint32_t bf = smem_u32(&bars[B_BFULL]);
                    mbar_expect_tx(bf, (uint32_t)(nkb * 2 * B_BYTES));
                    for (int kb = 0; kb < nkb; ++kb) {
                        tma_load_2d(smem_u32(b_hi(0, kb)), &tmDh, kb * KB, (int)d_row0, bf);
                        tma_load_2d(smem_u32(b_lo(0, kb)), &tmDl, kb * KB, (int)d_row0, bf);
                    }
                    seg_prev = I.seg;
                    ++nseg;
                }
                for (int kb = 0; kb < nkb; ++kb, ++q) {
                    const int s = (int)(q % NST);
                    const int64_t use = q / NST;
                    if (use > 0) mbar_wait(smem_u32(&bars[B_EMPTY + s]), (uint32_t)((use - 1) & 1));
                    const uint32_t full = smem_u32(&bars[s]);
                    mbar_expect_tx(full, RES ? A_BYTES : A_BYTES + 2 * B_BYTES);
                    tma_load_2d(smem_u32(a_hi(s)), &tmY, kb * KB, (int)row0, full);
                    if (!RES) {
                        tma_load_2d(smem_u32(b_hi(s, kb)), &tmDh, kb * KB, (int)d_row0, full);
                        tma_load_2d(smem_u32(b_lo(s, kb)), &tmDl, kb * KB, (int)d_row0, full);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) |
                               ((uint32_t)(TM >> 4) << 24);
        int64_t q = 0, n = 0, seg_prev = -1, nseg = 0;
        ItemWalk W(it0, it1, tile_start, P, nchunk);
        for (int64_t it = it0; it < it1; ++it, ++n, W.next(tile_start, P, nchunk)) {
            const Item I = W.I;
            const int b = (int)(n & 1);
            const int64_t buse = n >> 1;
            if (lane == 0) {
                if (RES && I.seg != seg_prev) {
                    mbar_wait(smem_u32(&bars[B_BFULL]), (uint32_t)(nseg & 1));
                    seg_prev = I.seg;
                    ++nseg;
                }
                if (buse > 0) mbar_wait(smem_u32(&bars[B_TEMPTY + b]), (uint32_t)((buse - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t tacc = tmem + (uint32_t)(b * TN);
                for (int kb = 0; kb < nkb; ++kb, ++q) {
                    const int s = (int)(q % NST);
                    mbar_wait(smem_u32(&bars[B_SPLIT + s]), (uint32_t)((q / NST) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint64_t dah = sw128_desc(smem_u32(a_hi(s)));
                    const uint64_t dal = sw128_desc(smem_u32(a_lo(s)));
                    const uint64_t dbh = sw128_desc(smem_u32(b_hi(s, kb)));
                    const uint64_t dbl = sw128_desc(smem_u32(b_lo(s, kb)));
#pragma unroll
                    for (int k = 0; k < KB / 8; ++k) {
                        const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);
                        const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
                        mma_tf32(tacc, dah + adv, dbh + adv, idesc, acc0);
                        mma_tf32(tacc, dah + adv, dbl + adv, idesc, 1u);
                        mma_tf32(tacc, dal + adv, dbh + adv, idesc, 1u);
                    }
                    mma_commit(smem_u32(&bars[B_EMPTY + s]));               // stage free
                    if (kb == nkb - 1) mma_commit(smem_u32(&bars[B_TFULL + b]));  // accumulator ready
                }
                if (RES) {  // resident D no longer needed after this item?
                    const bool last = (it + 1 >= it1) || W.seg_ends();
                    if (last) mma_commit(smem_u32(&bars[B_BFREE]));
                }
            }
            __syncwarp();
        }
    } else if ((warp >= 2 && warp < 6) || (CODE && warp >= 10)) {
        // ---------------- epilogue (TMEM lane quadrant = warp % 4): thread =
        // signal row; each 32x32 block is staged in smem and written by one
        // TMA store (async, full lines); quadrants straddling a shard end use
        // plain stores so rows of the next shard are never touched
        const int quad = warp & 3;
        const int half = warp >= 10 ? 1 : 0;
        float* stg = stg_base + (warp - 2) * 2 * 1024;     // !CODE only
        float* xch = stg_base + quad * 100;                // CODE: the quadrant pair's exchange slots
        float* diag = stg_base + 4 * 100 + quad * 256;     // CODE: lower warp's copy of the shard's G diagonal
        int diag_p = -1;
        const int c_mid = ((K + 63) / 64) * 32;
        int64_t n = 0;
        int sb = 0;  // staging buffer toggle
        ItemWalk W(it0, it1, tile_start, P, nchunk);
        for (int64_t it = it0; it < it1; ++it, ++n, W.next(tile_start, P, nchunk)) {
            const Item I = W.I;
            const int b = (int)(n & 1);
            // CODE: ||y||^2 of this warp's rows and the shard's G diagonal are
            // fetched before the accumulator is waited for (their latency then
            // overlaps the MMA instead of the epilogue)
            float ysq_pre = 0.0f;
            if constexpr (CODE) {
                if (half == 0) {
                    const int64_t r = off[I.p] + I.tile * TM + quad * 32 + lane;
                    if (r < off[I.p + 1]) ysq_pre = __ldg(s1.ysq + r);
                    if (diag_p != I.p) {
                        __syncwarp();
                        for (int k = lane; k < K; k += 32) diag[k] = __ldg(s1.G + ((int64_t)I.p * K + k) * K + k);
                        diag_p = I.p;
                        __syncwarp();
                    }
                }
            }
            mbar_wait(smem_u32(&bars[B_TFULL + b]), (uint32_t)((n >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t s_hi = off[I.p + 1];
            const int64_t row_base = off[I.p] + I.tile * TM + quad * 32;
            const int nrows = (int)max((int64_t)0, min((int64_t)32, s_hi - row_base));
            const int n0 = I.chunk * TN;
            const int ncols = min(TN, K - n0);
            const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * TN);
            if constexpr (CODE) {
                code_step1(s1, trow, row_base, nrows, I.p, K, half, half ? c_mid : 0, half ? K : min(c_mid, K),
                           xch, reinterpret_cast<uint32_t*>(xch + 32), reinterpret_cast<unsigned*>(xch + 64),
                           diag, ysq_pre, quad, alpha, lda, lane);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars[B_TEMPTY + b]));
                continue;
            }
            // one 32x32 block: TMA store from swizzled staging (conflict-free
            // 16-byte smem writes), or plain stores for a partial quadrant
            auto put = [&](const uint32_t (&v)[32], int c) {
                const int j0 = n0 + c;
                if (nrows == 32) {
                    float* buf = stg + sb * 1024;
                    // the TMA store issued two blocks ago must have read this buffer
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
                    float4* row4 = reinterpret_cast<float4*>(buf + lane * 32);
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq)
                        row4[qq ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * qq]), __uint_as_float(v[4 * qq + 1]),
                                                            __uint_as_float(v[4 * qq + 2]), __uint_as_float(v[4 * qq + 3]));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                (uint64_t)&tmA),
                            "r"(j0), "r"((int)row_base), "r"(smem_u32(buf))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    sb ^= 1;
                } else if (lane < nrows) {
                    float* out = alpha + (row_base + lane) * lda;
#pragma unroll
                    for (int qq = 0; qq < 32; ++qq)
                        if (j0 + qq < K) out[j0 + qq] = __uint_as_float(v[qq]);
                }
            };
            // TMEM loads run one block ahead of the stores
            uint32_t va[32], vb[32];
            tmem_ld32(va, trow);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll 1
            for (int c = 0; c < ncols; c += 64) {
                if (c + 32 < ncols) tmem_ld32(vb, trow + (uint32_t)(c + 32));
                put(va, c);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c + 32 >= ncols) break;
                if (c + 64 < ncols) tmem_ld32(va, trow + (uint32_t)(c + 64));
                put(vb, c + 32);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[B_TEMPTY + b]));
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    } else if (warp >= 6 && warp < 10) {
        // ---------------- 3xTF32 split of the Y k-block (warps 6-9)
        const int st = tid - 6 * 32;  // 0..127
        int64_t q = 0;
        for (int64_t it = it0; it < it1; ++it) {
            for (int kb = 0; kb < nkb; ++kb, ++q) {
                const int s = (int)(q % NST);
                mbar_wait(smem_u32(&bars[s]), (uint32_t)((q / NST) & 1));
                float4* ah = (float4*)a_hi(s);
                float4* al = (float4*)a_lo(s);
#pragma unroll
                for (int e = st; e < A_BYTES / 16; e += 128) {
                    const float4 v = ah[e];
                    float4 h, l;
                    h.x = tf32_rna(v.x); l.x = v.x - h.x;
                    h.y = tf32_rna(v.y); l.y = v.y - h.y;
                    h.z = tf32_rna(v.z); l.z = v.z - h.z;
                    h.w = tf32_rna(v.w); l.w = v.w - h.w;
                    ah[e] = h;
                    al[e] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars[B_SPLIT + s]));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TN));
}

// tile_start[p] = first 128-signal tile of shard p (prefix over shards)
__global__ void k_tile_layout(const int64_t* __restrict__ off, int P, int64_t* __restrict__ ts,
                              int* __restrict__ zero) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (zero) { zero[0] = 0; zero[1] = 0; }   // CODE: deferred count, deferred-OMP work counter
        int64_t t = 0;
        for (int p = 0; p < P; ++p) {
            ts[p] = t;
            t += (off[p + 1] - off[p] + TM - 1) / TM;
        }
        ts[P] = t;
    }
}

// D (P*K rows of m fp32, atom-major) -> D_hi, D_lo (P*K rows of m_pad, zero padded)
__global__ void k_split_dict(int64_t rows, int m, int m_pad, const float* __restrict__ D,
                             float* __restrict__ Dh, float* __restrict__ Dl) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * m_pad) return;
    const int64_t r = e / m_pad;
    const int c = (int)(e % m_pad);
    const float x = c < m ? D[r * m + c] : 0.0f;
    const float h = tf32_rna(x);
    Dh[e] = h;
    Dl[e] = x - h;
}

// ---------------------------------------------------------------- host side
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn g_encode = nullptr;
std::once_flag g_once;

void load_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = (EncodeFn)fn;
}

bool make_map_plain(CUtensorMap* map, const float* ptr, int64_t cols, int64_t rows, int64_t ld_elems) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* map, const float* ptr, int64_t cols, int64_t rows, int64_t ld_elems,
              int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {(cuuint32_t)KB, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// 2-D fp32 tensor map with 128-byte swizzle for the other tcgen05 kernels
// (box: box_cols fp32 columns = 128 bytes, box_rows rows)
bool tc_map_f32(CUtensorMap* map, const float* ptr, int64_t cols, int64_t rows, int64_t ld_elems,
                int box_rows) {
    std::call_once(g_once, load_encode);
    return g_encode != nullptr && make_map(map, ptr, cols, rows, ld_elems, box_rows);
}

int64_t corr_tc_ws_bytes(int P, int64_t m, int64_t K) {
    const int64_t m_pad = (m + KB - 1) / KB * KB;
    return 2 * (int64_t)P * K * m_pad * 4 + 256 + 8 * ((int64_t)P + 1) + 256;
}

static int corr_tc_launch(int64_t N, const float* Y, int64_t ldy, const int64_t* off, int P,
                          const float* D, int64_t m, int64_t K, float* alpha, int64_t lda, void* ws,
                          int64_t ws_bytes, const Step1* s1, cudaStream_t st) {
    std::call_once(g_once, load_encode);
    if (!g_encode || ws == nullptr || ws_bytes < corr_tc_ws_bytes(P, m, K)) return (int)cudaErrorNotSupported;
    if ((ldy * 4) % 16 != 0 || ((uintptr_t)Y & 15) != 0) return (int)cudaErrorNotSupported;
    const int64_t m_pad = (m + KB - 1) / KB * KB;
    float* Dh = (float*)ws;
    float* Dl = Dh + (int64_t)P * K * m_pad;
    const int64_t rows = (int64_t)P * K;
    k_split_dict<<<(unsigned)((rows * m_pad + 255) / 256), 256, 0, st>>>(rows, (int)m, (int)m_pad, D, Dh, Dl);
    // the Y map spans all N rows: tiles past a shard's end read neighbouring
    // signals (never stored), past N the TMA zero-fills
    CUtensorMap mY, mDh, mDl;
    CUtensorMap mA;
    if (!make_map(&mY, Y, m, N, ldy, TM) || !make_map(&mDh, Dh, m_pad, rows, m_pad, TN) ||
        !make_map(&mDl, Dl, m_pad, rows, m_pad, TN) || (lda * 4) % 16 != 0 ||
        ((uintptr_t)alpha & 15) != 0 || !make_map_plain(&mA, alpha, K, N, lda))
        return (int)cudaErrorNotSupported;
    int n_sm = 148;
    {
        cudaError_t e = set_max_smem((const void*)k_corr_tc2<true, false>, Cfg<true, false>::SMEM);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_corr_tc2<false, false>, Cfg<false, false>::SMEM);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_corr_tc2<true, true>, Cfg<true, true>::SMEM);
        if (e == cudaSuccess) e = set_max_smem((const void*)k_corr_tc2<false, true>, Cfg<false, true>::SMEM);
        if (e != cudaSuccess) return (int)e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    int64_t* tile_start = (int64_t*)((unsigned char*)ws + 2 * (int64_t)P * K * m_pad * 4 + 256);
    tile_start = (int64_t*)(((uintptr_t)tile_start + 255) & ~(uintptr_t)255);
    k_tile_layout<<<1, 32, 0, st>>>(off, P, tile_start, s1 ? s1->n_deferred : nullptr);
    const int nchunk = (int)((K + TN - 1) / TN);
    // upper bound on work items (the kernel reads the exact count on device)
    const int64_t max_items = ((N + TM - 1) / TM + P) * nchunk;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(n_sm, max_items));
    const int nkb = (int)(m_pad / KB);
    const Step1 sv = s1 ? *s1 : Step1{};
    auto fn = nkb <= RES_KB ? (s1 ? k_corr_tc2<true, true> : k_corr_tc2<true, false>)
                            : (s1 ? k_corr_tc2<false, true> : k_corr_tc2<false, false>);
    const int smem = nkb <= RES_KB ? (s1 ? Cfg<true, true>::SMEM : Cfg<true, false>::SMEM)
                                   : (s1 ? Cfg<false, true>::SMEM : Cfg<false, false>::SMEM);
    fn<<<grid, NWARP2 * 32, smem, st>>>(mY, mDh, mDl, mA, off, tile_start, P, (int)K, nkb, nchunk,
                                               alpha, lda, sv);
    return (int)cudaGetLastError();
}

int correlate_tc_f32(int64_t N, const float* Y, int64_t ldy, const int64_t* off, int64_t max_rows,
                     int P, const float* D, int64_t m, int64_t K, float* alpha, int64_t lda, void* ws,
                     int64_t ws_bytes, cudaStream_t st) {
    return corr_tc_launch(N, Y, ldy, off, P, D, m, K, alpha, lda, ws, ws_bytes, nullptr, st);
}

int code_step1_tc_f32(int64_t N, const float* Y, int64_t ldy, const int64_t* off, int P, const float* D,
                      int64_t m, int64_t K, float* alpha, int64_t lda, void* ws, int64_t ws_bytes,
                      const float* ysq, const float* G, float eps, float guard, int cap, int32_t* idx,
                      float* val, int32_t* counts, int8_t* status, float* gap, int* n_deferred, cudaStream_t st) {
    if (K > TN || N > 0x7fffffffll || cap < 1) return (int)cudaErrorNotSupported;
    Step1 s1;
    s1.ysq = ysq; s1.G = G; s1.eps2 = eps * eps; s1.guard = guard; s1.cap = cap;
    s1.idx = idx; s1.val = val; s1.counts = counts; s1.status = status;
    s1.n_deferred = n_deferred;
    s1.gap = gap;

    return corr_tc_launch(N, Y, ldy, off, P, D, m, K, alpha, lda, ws, ws_bytes, &s1, st);
}

}  // namespace sdb
