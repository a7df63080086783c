// 64x64x64 FP64 tile GEMM in shared memory, 256 threads: SIMT 4x4 micro-tiles
// (the clustered solver's tile_mm) vs warp-level DMMA m8n8k4.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
constexpr int CB = 64, CBP = 65;
__device__ __forceinline__ void mm_simt(const double* Xs, const double* Ys, double acc[16]) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    for (int q = 0; q < CB; ++q) {
        double xv[4], yv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = Xs[(ty + 16 * a) * CBP + q];
#pragma unroll
        for (int b = 0; b < 4; ++b) yv[b] = Ys[(tx + 16 * b) * CBP + q];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a * 4 + b] = fma(xv[a], yv[b], acc[a * 4 + b]);
    }
}
__device__ __forceinline__ void mm_dmma(const double* Xs, const double* Ys, double acc[16]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r0 = 16 * (w >> 1), c0 = 32 * (w & 1);
    const int ar = lane >> 2, ak = lane & 3;
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < CB; k0 += 4) {
        double a[2], b[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) a[mt] = Xs[(r0 + 8 * mt + ar) * CBP + k0 + ak];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) b[nt] = Ys[(c0 + 8 * nt + ar) * CBP + k0 + ak];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                double* c = &acc[(mt * 4 + nt) * 2];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[0]), "+d"(c[1]) : "d"(a[mt]), "d"(b[nt]));
            }
    }
}
template <bool DM>
__global__ void kg(const double* X, const double* Y, double* C, long long* cyc, int reps) {
    extern __shared__ double gsm[];
    double* Xs = gsm;
    double* Ys = gsm + CB * CBP;
    for (int e = threadIdx.x; e < CB * CB; e += 256) { Xs[(e / CB) * CBP + e % CB] = X[e]; Ys[(e / CB) * CBP + e % CB] = Y[e]; }
    __syncthreads();
    double acc[16];
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        long long t0 = clock64();
        if (DM) mm_dmma(Xs, Ys, acc); else mm_simt(Xs, Ys, acc);
        __syncthreads();
        long long t1 = clock64();
        best = min(best, t1 - t0);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    for (int i = 0; i < 16; ++i) {
        int r, c;
        if (DM) { const int t = i >> 1, mt = t >> 2, nt = t & 3; r = 16 * (w >> 1) + 8 * mt + (lane >> 2); c = 32 * (w & 1) + 8 * nt + 2 * (lane & 3) + (i & 1); }
        else { r = ty + 16 * (i >> 2); c = tx + 16 * (i & 3); }
        C[r * CB + c] = acc[i];
    }
    if (threadIdx.x == 0) cyc[0] = best;
}
int main() {
    std::vector<double> X(CB * CB), Y(CB * CB), ref(CB * CB);
    for (int i = 0; i < CB * CB; ++i) { X[i] = sin(i * 0.37); Y[i] = cos(i * 0.11); }
    for (int r = 0; r < CB; ++r) for (int c = 0; c < CB; ++c) { double s = 0; for (int q = 0; q < CB; ++q) s += X[r * CB + q] * Y[c * CB + q]; ref[r * CB + c] = s; }
    double *dX, *dY, *dC; long long* dc;
    cudaMalloc(&dX, 8 * CB * CB); cudaMalloc(&dY, 8 * CB * CB); cudaMalloc(&dC, 8 * CB * CB); cudaMalloc(&dc, 8);
    cudaMemcpy(dX, X.data(), 8 * CB * CB, cudaMemcpyHostToDevice); cudaMemcpy(dY, Y.data(), 8 * CB * CB, cudaMemcpyHostToDevice);
    std::vector<double> C(CB * CB); long long cy;
    const int smem = 2 * CB * CBP * 8;
    cudaFuncSetAttribute(kg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kg<false><<<1, 256, smem>>>(dX, dY, dC, dc, 5); cudaDeviceSynchronize();
    cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(C.data(), dC, 8 * CB * CB, cudaMemcpyDeviceToHost);
    double e = 0; for (int i = 0; i < CB * CB; ++i) e = fmax(e, fabs(C[i] - ref[i]));
    printf("simt: %lld cycles, max err %.2e\n", cy, e);
    kg<true><<<1, 256, smem>>>(dX, dY, dC, dc, 5); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(C.data(), dC, 8 * CB * CB, cudaMemcpyDeviceToHost);
    e = 0; for (int i = 0; i < CB * CB; ++i) e = fmax(e, fabs(C[i] - ref[i]));
    printf("dmma: %lld cycles, max err %.2e\n", cy, e);
}
