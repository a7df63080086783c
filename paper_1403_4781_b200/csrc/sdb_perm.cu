// Device side of the split permutation (trainer.split_indices,
// trainer.py:208-209: numpy.random.default_rng(seed).permutation(N)).
//
// The host parses the PCG64 stream into the Fisher-Yates swap targets j_k
// (step k swaps positions i_k = n-1-k and j_k <= i_k; sdb_pcg64_swap_targets);
// the sequential swap loop is then resolved here in parallel, exactly:
//   last[v] = the last step whose target is v, prev(k) = the previous step
//   with the same target as step k (one stable radix sort of (j_k, k));
//   u_k, the value moved out of position i_k by step k, is the value step
//   M(k) moved into i_k, where M(k) = last[i_k] (or prev(k) when j_k = i_k,
//   since every step targeting i_k comes no later than k); a chain
//   k -> M(k) -> ... ends at a step whose position was never written, whose
//   value is its own index i;
//   final[i_k] = u_{prev(k)} (or j_k if no earlier step targeted j_k), and
//   final[0] = u_{last[0]} (or 0).
// Chains are short (mean ~1, max ~22 at n = 2M), so each thread walks its own.
#include <cub/device/device_radix_sort.cuh>

#include "sdb_common.cuh"

namespace sdb {

namespace {
struct PermWs {
    uint32_t *keys_out, *vals_in, *vals_out, *u;
    int32_t *prev, *last, *M;
    void* cub_tmp;
    size_t cub_bytes;
    unsigned char* end;
};

int key_bits(int64_t n) {
    int b = 1;
    while (b < 32 && ((int64_t)1 << b) < n) ++b;
    return b;
}

PermWs carve(void* base, int64_t n) {
    const int64_t S = n - 1;
    PermWs w{};
    unsigned char* p = (unsigned char*)base;
    auto take = [&](int64_t bytes) { void* r = p; p += (bytes + 255) & ~int64_t(255); return r; };
    w.keys_out = (uint32_t*)take(4 * S);
    w.vals_in = (uint32_t*)take(4 * S);
    w.vals_out = (uint32_t*)take(4 * S);
    w.u = (uint32_t*)take(4 * S);
    w.prev = (int32_t*)take(4 * S);
    w.M = (int32_t*)take(4 * S);
    w.last = (int32_t*)take(4 * n);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)S, 0, key_bits(n));
    w.cub_bytes = tb;
    w.cub_tmp = take((int64_t)tb);
    w.end = p;
    return w;
}
}  // namespace

__global__ void k_fy_iota(int64_t S, uint32_t* __restrict__ v) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < S) v[k] = (uint32_t)k;
}

__global__ void k_fy_links(int64_t S, const uint32_t* __restrict__ key, const uint32_t* __restrict__ step,
                           int32_t* __restrict__ prev, int32_t* __restrict__ last) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= S) return;
    const uint32_t kv = key[t], st = step[t];
    prev[st] = (t > 0 && key[t - 1] == kv) ? (int32_t)step[t - 1] : -1;
    if (t == S - 1 || key[t + 1] != kv) last[kv] = (int32_t)st;
}

__global__ void k_fy_moves(int64_t S, int64_t n, const uint32_t* __restrict__ js, const int32_t* __restrict__ prev,
                           const int32_t* __restrict__ last, int32_t* __restrict__ M) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    const int64_t i = n - 1 - k;
    M[k] = ((int64_t)js[k] == i) ? prev[k] : last[i];
}

__global__ void k_fy_resolve(int64_t S, int64_t n, const int32_t* __restrict__ M, uint32_t* __restrict__ u) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    int64_t x = k;
    for (int32_t y = M[x]; y >= 0; y = M[x]) x = y;
    u[k] = (uint32_t)(n - 1 - x);
}

__global__ void k_fy_final(int64_t S, int64_t n, const uint32_t* __restrict__ js, const int32_t* __restrict__ prev,
                           const int32_t* __restrict__ last, const uint32_t* __restrict__ u,
                           int64_t* __restrict__ perm) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    const int32_t pk = prev[k];
    perm[n - 1 - k] = pk >= 0 ? (int64_t)u[pk] : (int64_t)js[k];
    if (k == 0) {
        const int32_t l0 = last[0];
        perm[0] = l0 >= 0 ? (int64_t)u[l0] : 0;
    }
}

int64_t perm_ws_bytes(int64_t n) {
    if (n < 2) return 256;
    PermWs w = carve(nullptr, n);
    return (int64_t)(w.end - (unsigned char*)nullptr) + 256;
}

int perm_from_targets(int64_t n, const uint32_t* js, int64_t* perm, void* ws, int64_t ws_bytes,
                      cudaStream_t st) {
    if (n == 1) return (int)cudaMemsetAsync(perm, 0, sizeof(int64_t), st);
    const int64_t S = n - 1;
    PermWs w = carve(ws, n);
    if ((int64_t)(w.end - (unsigned char*)ws) > ws_bytes) return (int)cudaErrorInvalidValue;
    const unsigned g = (unsigned)((S + 255) / 256);
    k_fy_iota<<<g, 256, 0, st>>>(S, w.vals_in);
    size_t tb = w.cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, js, w.keys_out, w.vals_in, w.vals_out,
                                                    (int)S, 0, key_bits(n), st);
    if (e != cudaSuccess) return (int)e;
    cudaMemsetAsync(w.last, 0xff, sizeof(int32_t) * n, st);
    k_fy_links<<<g, 256, 0, st>>>(S, w.keys_out, w.vals_out, w.prev, w.last);
    k_fy_moves<<<g, 256, 0, st>>>(S, n, js, w.prev, w.last, w.M);
    k_fy_resolve<<<g, 256, 0, st>>>(S, n, w.M, w.u);
    k_fy_final<<<g, 256, 0, st>>>(S, n, js, w.prev, w.last, w.u, perm);
    return (int)cudaGetLastError();
}

}  // namespace sdb
