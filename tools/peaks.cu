// Roofline denominators the driver's MEASURED_PEAKS.json does not carry,
// measured on the box by bench.py ("TF32, FP32-SIMT and L2
// bandwidth peaks are not measured there; measure them before quoting
// fractions"). Measurement harness only (not product code):
//   peak_fma_f32: FP32 FFMA throughput (8 independent chains per thread,
//                 one wave of 148 x 8 CTAs of 256 threads)
//   peak_l2_read: L2 read bandwidth (float4 .cg loads, buffer well below L2,
//                 the grid sweeps it `passes` times after a warm-up launch)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared
//        -Xcompiler -fPIC -o tools/_lat/libpeaks.so tools/peaks.cu
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_fma(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void k_l2(const float4* __restrict__ buf, int64_t n4, int passes, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        for (int64_t k = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; k < n4; k += stride) {
            const float4 v = __ldcg(buf + k);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.678f) out[0] = acc.x;
}

static float time_ms(void (*launch)(void*), void* ctx) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(ctx);  // warm-up
    cudaEventRecord(a);
    launch(ctx);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

struct FmaCtx { float* out; int blocks, iters; };
struct L2Ctx { const float4* buf; int64_t n4; int blocks, passes; float* out; };

extern "C" {

// FP32 FFMA TFLOP/s (2 flops per FMA)
double peak_fma_f32(void) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    FmaCtx c{nullptr, sms * 8, 4096};
    cudaMalloc(&c.out, sizeof(float) * c.blocks);
    const float ms = time_ms([](void* p) {
        FmaCtx* c = (FmaCtx*)p;
        k_fma<<<c->blocks, 256>>>(c->out, c->iters, 0.999f, 0.001f);
    }, &c);
    cudaFree(c.out);
    const double flops = 2.0 * 8 * 16 * (double)c.iters * 256 * c.blocks;
    return flops / (ms * 1e-3) / 1e12;
}

// L2 read GB/s over a buffer of `bytes` (should be well below the L2 size)
double peak_l2_read(int64_t bytes) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    L2Ctx c{};
    c.n4 = bytes / 16;
    c.blocks = sms * 4;
    c.passes = 20;
    float4* buf = nullptr;
    cudaMalloc(&buf, c.n4 * 16);
    cudaMemset(buf, 0, c.n4 * 16);
    cudaMalloc(&c.out, sizeof(float));
    c.buf = buf;
    const float ms = time_ms([](void* p) {
        L2Ctx* c = (L2Ctx*)p;
        k_l2<<<c->blocks, 512>>>(c->buf, c->n4, c->passes, c->out);
    }, &c);
    cudaFree(buf);
    cudaFree(c.out);
    return (double)c.n4 * 16 * c.passes / (ms * 1e-3) / 1e9;
}
}
