// standalone timing of factor_inverse on one 64x64 SPD tile (256 threads)
#include "../../paper_1403_4781_b200/csrc/sdb_chol.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace sdb;
__global__ void kf(const double* A, double* T, long long* cyc, int reps) {
    extern __shared__ double xs[];
    __shared__ __align__(16) double fring[FNB * FSLOT];
    __shared__ uint64_t fbars[2 * FNB];
    __shared__ double fdval[CB];
    __shared__ int8_t sdep[CB];
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
        for (int e = threadIdx.x; e < CB * CB; e += 256) xs[(e / CB) * CBP + e % CB] = A[e];
        __syncthreads();
        long long t0 = clock64();
        factor_inverse(xs, CB, 1e-12, fring, fbars, fdval, sdep);
        __syncthreads();
        long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    for (int e = threadIdx.x; e < CB * CB; e += 256) T[e] = xs[(e / CB) * CBP + e % CB];
    if (threadIdx.x == 0) cyc[0] = best;
}
int main() {
    std::vector<double> M(CB * CB), A(CB * CB, 0.0);
    srand(1);
    for (auto& v : M) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < CB; ++i) for (int j = 0; j < CB; ++j) { double s = 0; for (int k = 0; k < CB; ++k) s += M[i*CB+k] * M[j*CB+k]; A[i*CB+j] = s + (i == j ? 1.0 : 0.0); }
    double *dA, *dT; long long* dc;
    cudaMalloc(&dA, 8 * CB * CB); cudaMalloc(&dT, 8 * CB * CB); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), 8 * CB * CB, cudaMemcpyHostToDevice);
    kf<<<1, 256, CB * CBP * 8>>>(dA, dT, dc, 5);
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    std::vector<double> T(CB * CB); cudaMemcpy(T.data(), dT, 8 * CB * CB, cudaMemcpyDeviceToHost);
    // check T A T^T = I
    double err = 0;
    for (int i = 0; i < CB; ++i) for (int j = 0; j < CB; ++j) {
        double s = 0;
        for (int a = 0; a < CB; ++a) for (int b = 0; b < CB; ++b) s += T[i*CB+a] * A[a*CB+b] * T[j*CB+b];
        err = fmax(err, fabs(s - (i == j)));
    }
    {   // host reference T = L^-1
        std::vector<double> L(CB * CB, 0.0), Ti(CB * CB, 0.0);
        for (int j = 0; j < CB; ++j) {
            double s = A[j*CB+j]; for (int q = 0; q < j; ++q) s -= L[j*CB+q] * L[j*CB+q];
            L[j*CB+j] = sqrt(s);
            for (int i = j + 1; i < CB; ++i) { double t = A[i*CB+j]; for (int q = 0; q < j; ++q) t -= L[i*CB+q] * L[j*CB+q]; L[i*CB+j] = t / L[j*CB+j]; }
        }
        for (int c = 0; c < CB; ++c) for (int r = 0; r < CB; ++r) {
            double t = (r == c); for (int q = 0; q < r; ++q) t -= L[r*CB+q] * Ti[q*CB+c];
            Ti[r*CB+c] = t / L[r*CB+r];
        }
        int shown = 0;
        for (int r = 0; r < CB && shown < 6; ++r) for (int q = 0; q < CB && shown < 6; ++q)
            if (fabs(T[r*CB+q] - Ti[r*CB+q]) > 1e-9 * (1 + fabs(Ti[r*CB+q]))) { printf("  T[%d][%d] gpu %.6g ref %.6g\n", r, q, T[r*CB+q], Ti[r*CB+q]); ++shown; }
    }
    printf("factor_inverse: %lld cycles (%.1f per column), |T A T^T - I| = %.2e\n", c, c / 64.0, err);
}
