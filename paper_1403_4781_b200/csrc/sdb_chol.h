// Shard-batched FP64 blocked Cholesky solve (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sdb {
int64_t chol_ws_bytes(int P, int K);
// Solves A Z = B in place on B for every shard; A is overwritten by L.
// wsq (optional, P): ||L^-1 B||_F^2 = <Z, B>, the explained energy, so the
// least-squares residual is ||Y||^2 - wsq.
int chol_solve(int P, int K, int m, double* A, double* B, const int32_t* usage, double rel_tol,
               int8_t* depmask, int32_t* ndep, double* wsq, void* ws, cudaStream_t st);
}  // namespace sdb
