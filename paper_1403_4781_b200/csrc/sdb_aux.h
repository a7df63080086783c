// Patch pipeline / data-movement launch interface (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sdb {
template <typename T>
int gather_rows(int64_t rows, int m, const T* in, int64_t ldi, const int64_t* perm, T* out, int64_t ldo,
                cudaStream_t st);
template <typename T>
int ingest_gather(int64_t rows, int m, const double* src, int64_t ldi, const int64_t* perm, T* out, int64_t ldo,
                  int32_t* bad, cudaStream_t st, const double* dsrc = nullptr, int64_t drows = 0);
template <typename T>
int csc_to_codes(int64_t N, int cap, const int64_t* indptr, const int64_t* indices, const double* data,
                 int32_t* idx, T* val, int32_t* counts, cudaStream_t st);
int normalize_rows(int64_t rows, int m, const double* in, double* out, double* scales, cudaStream_t st);
template <typename T>
int extract_patches(const double* img, int H, int W, int p, int s, T* out, cudaStream_t st);
template <typename T>
int reconstruct(int H, int W, int p, int s, const double* D, int cap, const int32_t* idx, const T* val,
                const int32_t* counts, double lo, double hi, double* out, cudaStream_t st);
int reconstruct_dense(int H, int W, int p, int s, const double* P, double* out, cudaStream_t st);
}  // namespace sdb
