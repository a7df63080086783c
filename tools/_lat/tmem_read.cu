// TMEM read microbenchmark: how fast can the signal warps sweep a 128 x 512 fp32
// accumulator (one k_omp_tc scan)? Separates tcgen05.ld latency from TMEM read
// bandwidth: 4 or 8 warps, x32 / x64 / x16 shapes, 1..4 loads in flight, with the
// kernel's |.|-max reduction or a 1-instruction consumer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_read tmem_read.cu && ./tmem_read
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1403_4781_b200/csrc/sdb_tc.cuh"
using namespace sdb;

__device__ __forceinline__ void tmem_ld16(uint32_t (&v)[16], uint32_t taddr) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

template <int N, bool HEAVY>
__device__ __forceinline__ float eat(const uint32_t (&v)[N], float acc) {
    if (HEAVY) {
        float m0 = 0.f, m1 = 0.f;
#pragma unroll
        for (int t = 0; t < N; t += 2) {
            m0 = fmaxf(m0, fabsf(__uint_as_float(v[t])));
            m1 = fmaxf(m1, fabsf(__uint_as_float(v[t + 1])));
        }
        return fmaxf(acc, fmaxf(m0, m1));
    } else {
        return acc + __uint_as_float(v[0] ^ v[N - 1]);
    }
}

// MODE 0: x32, ld-wait-eat; 1: x32 double buffered (kernel pattern); 2: x32 two loads then one wait;
// 3: x64 ld-wait-eat; 4: x16 four loads then one wait; 5: x16 rolling 4 in flight (wait each time)
template <int MODE, bool HEAVY>
__global__ void __launch_bounds__(256, 1) k(int reps, long long* out, float* sink) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {
            uint32_t v[32];
#pragma unroll 1
            for (int b = 0; b < 16; ++b) { tmem_ld32(v, trow + b * 32); tmem_wait_ld(); acc = eat<32, HEAVY>(v, acc); }
        } else if (MODE == 1) {
            uint32_t va[32], vb[32];
            tmem_ld32(va, trow);
#pragma unroll
            for (int b = 0; b < 16; b += 2) {
                tmem_wait_ld();
                tmem_ld32(vb, trow + (b + 1) * 32);
                acc = eat<32, HEAVY>(va, acc);
                tmem_wait_ld();
                if (b + 2 < 16) tmem_ld32(va, trow + (b + 2) * 32);
                acc = eat<32, HEAVY>(vb, acc);
            }
        } else if (MODE == 2) {
            uint32_t va[32], vb[32];
#pragma unroll 1
            for (int b = 0; b < 16; b += 2) {
                tmem_ld32(va, trow + b * 32);
                tmem_ld32(vb, trow + (b + 1) * 32);
                tmem_wait_ld();
                acc = eat<32, HEAVY>(va, acc);
                acc = eat<32, HEAVY>(vb, acc);
            }
        } else if (MODE == 3) {
            uint32_t va[32], vb[32];
#pragma unroll 1
            for (int b = 0; b < 16; b += 2) {
                tmem_ld64(va, vb, trow + b * 32);
                tmem_wait_ld();
                acc = eat<32, HEAVY>(va, acc);
                acc = eat<32, HEAVY>(vb, acc);
            }
        } else if (MODE == 4) {
            uint32_t v0[16], v1[16], v2[16], v3[16];
#pragma unroll 1
            for (int b = 0; b < 32; b += 4) {
                tmem_ld16(v0, trow + b * 16);
                tmem_ld16(v1, trow + (b + 1) * 16);
                tmem_ld16(v2, trow + (b + 2) * 16);
                tmem_ld16(v3, trow + (b + 3) * 16);
                tmem_wait_ld();
                acc = eat<16, HEAVY>(v0, acc);
                acc = eat<16, HEAVY>(v1, acc);
                acc = eat<16, HEAVY>(v2, acc);
                acc = eat<16, HEAVY>(v3, acc);
            }
        } else if (MODE == 5) {
            // 8 x32 loads issued back to back into 8 register buffers is too many registers;
            // x32 with 3 buffers: two loads always in flight behind the one being eaten
            uint32_t va[32], vb[32], vc[32];
            tmem_ld32(va, trow);
            tmem_ld32(vb, trow + 32);
#pragma unroll
            for (int b = 0; b < 15; b += 3) {
                tmem_wait_ld();   // waits for both
                tmem_ld32(vc, trow + (b + 2) * 32);
                acc = eat<32, HEAVY>(va, acc);
                acc = eat<32, HEAVY>(vb, acc);
                tmem_wait_ld();
                tmem_ld32(va, trow + (b + 3) * 32);
                if (b + 4 < 16) tmem_ld32(vb, trow + (b + 4) * 32);
                acc = eat<32, HEAVY>(vc, acc);
            }
            tmem_wait_ld();
            acc = eat<32, HEAVY>(va, acc);
        }
    }
    tmem_fence_before();
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE, bool HEAVY>
void run(const char* name, int threads) {
    long long* out;
    float* sink;
    cudaMalloc(&out, 8 * 148);
    cudaMalloc(&sink, 4 * 148 * 256);
    const int reps = 2000;
    k<MODE, HEAVY><<<1, threads>>>(10, out, sink);
    k<MODE, HEAVY><<<1, threads>>>(reps, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / reps;
    printf("%-34s warps=%d %s  cycles/sweep(128x512 per 4 warps)=%8.1f  B/cyc=%6.1f  %s\n", name, threads / 32,
           HEAVY ? "absmax" : "light ", per, (threads / 128) * 128.0 * 512 * 4 / per,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(sink);
}

int main() {
    for (int th : {128, 256}) {
        run<0, false>("x32 ld-wait-eat", th);
        run<0, true>("x32 ld-wait-eat", th);
        run<1, false>("x32 double-buffered (kernel)", th);
        run<1, true>("x32 double-buffered (kernel)", th);
        run<2, false>("x32 two loads, one wait", th);
        run<2, true>("x32 two loads, one wait", th);
        run<3, false>("x64 ld-wait-eat", th);
        run<3, true>("x64 ld-wait-eat", th);
        run<4, false>("x16 four loads, one wait", th);
        run<4, true>("x16 four loads, one wait", th);
        run<5, false>("x32 three buffers", th);
        run<5, true>("x32 three buffers", th);
    }
    return 0;
}
