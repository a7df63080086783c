// Host memory experiment: permuted gather of N rows of m f64 + cast to f32
// with T threads (what a host-side conversion before PCIe would cost).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>
#include <algorithm>
int main(int argc, char** argv) {
    const int64_t N = 2040200, m = 64;
    const int T = argc > 1 ? atoi(argv[1]) : 16;
    std::vector<double> Y(N * m);
    for (int64_t i = 0; i < N * m; ++i) Y[i] = (double)(i % 1000) * 0.5;
    std::vector<int64_t> perm(N);
    for (int64_t i = 0; i < N; ++i) perm[i] = i;
    std::mt19937_64 rng(1);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<float> out(N * m);
    for (int rep = 0; rep < 4; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t]() {
                const int64_t lo = N * t / T, hi = N * (t + 1) / T;
                for (int64_t r = lo; r < hi; ++r) {
                    const double* s = &Y[perm[r] * m];
                    float* d = &out[r * m];
                    for (int k = 0; k < m; ++k) d[k] = (float)s[k];
                }
            });
        for (auto& x : th) x.join();
        auto t1 = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        printf("threads %d: %.2f ms  (%.1f GB/s read)\n", T, ms, N * m * 8 / ms / 1e6);
    }
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    return (int)out[12345] & 1;
}
