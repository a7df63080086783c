// Shared device helpers for the sparsedict-B200 kernels (sm_100a).
//
// Two arithmetic modes share every kernel template:
//   T = double : "exact" mode. Every product and sum is rounded separately
//                (__dmul_rn/__dadd_rn/__dsub_rn, no FMA contraction) and
//                loops keep the reference's iteration order, so the OMP
//                results are bitwise identical to the reference's Numba
//                kernels (_kernels.py), which LLVM compiles without FMA.
//   T = float  : "fast" mode. FP32 with FMA and warp-parallel reductions;
//                parity is tolerance-based.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#include <unordered_map>

#define SDB_WARP 32
#define SDB_FULL 0xffffffffu

namespace sdb {

template <typename T> struct Ar;

template <> struct Ar<double> {
    static constexpr bool kExact = true;
    __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
    // acc + a*b with two roundings (the reference's `acc += a * b`)
    __device__ __forceinline__ static double mac(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
    // acc - a*b with two roundings (the reference's `acc -= a * b`)
    __device__ __forceinline__ static double msub(double acc, double a, double b) {
        return __dsub_rn(acc, __dmul_rn(a, b));
    }
    __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
    __device__ __forceinline__ static double sqrt_(double a) { return __dsqrt_rn(a); }
};

template <> struct Ar<float> {
    static constexpr bool kExact = false;
    __device__ __forceinline__ static float mul(float a, float b) { return a * b; }
    __device__ __forceinline__ static float add(float a, float b) { return a + b; }
    __device__ __forceinline__ static float sub(float a, float b) { return a - b; }
    __device__ __forceinline__ static float mac(float acc, float a, float b) { return fmaf(a, b, acc); }
    __device__ __forceinline__ static float msub(float acc, float a, float b) { return fmaf(-a, b, acc); }
    __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
    __device__ __forceinline__ static float sqrt_(float a) { return __fsqrt_rn(a); }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SDB_FULL, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(SDB_FULL, v, o));
    return v;
}

__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(SDB_FULL, v, o));
    return v;
}

// Shard of signal i given the (P+1)-entry offsets array (binary search).
__device__ __forceinline__ int shard_of(const int64_t* __restrict__ off, int P, int64_t i) {
    int lo = 0, hi = P - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device
// context: cache the largest size already set per (kernel, device) so a
// process driving several GPUs sets it on each of them.
inline cudaError_t set_max_smem(const void* fn, int smem) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t key = ((uint64_t)(uintptr_t)fn << 8) ^ (uint64_t)dev;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= smem) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) done[key] = smem;
    return e;
}

}  // namespace sdb
