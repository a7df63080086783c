#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double sm[256];
    double x = out[threadIdx.x] + 1.0;
    float f = (float)x;
    sm[threadIdx.x] = x;
    __syncthreads();
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * 0.9999999;
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // F2F f64->f32->f64 + MUFU rsqrt chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = (double)rsqrtf((float)x) + 0.5;
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // FFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) f = fmaf(f, 0.9999f, 1e-6f);
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // LDS chain (dependent address)
    int idx = threadIdx.x & 1;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = ((int)sm[idx] + idx + 1) & 255;
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // barrier chain (all 256 threads)
    t0 = clock64();
    for (int i = 0; i < n; ++i) { sm[(threadIdx.x + i) & 255] = x; __syncthreads(); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
    // barrier + LDS + DMUL + STS chain (publish/consume)
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (threadIdx.x == (i & 255)) sm[i & 1] = x;
        __syncthreads();
        x = sm[i & 1] * 0.999;
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
    // double rsqrt (libdevice)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5;
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
    out[threadIdx.x] = x + f + idx;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64 * 8); cudaMemset(o, 0, 2048);
    int n = 1000;
    k<<<1, 256>>>(o, c, n); printf("e1 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    k<<<1, 256>>>(o, c, n); printf("e2 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* nm[8] = {"DFMA", "DMUL", "f2f+mufu.rsq+f2f+dadd", "FFMA", "LDS chain", "bar.sync(256)", "pub+bar+LDS+DMUL", "rsqrt(double)"};
    for (int i = 0; i < 8; ++i) printf("%-26s %.1f cycles/iter\n", nm[i], (double)h[i] / n);
    return 0;
}
