// tcgen05 3xTF32 correlation GEMM (placeholder until the tensor-core path lands).
#include "sdb_internal.h"

namespace sdb {
int correlate_tc_f32(const float*, int64_t, const int64_t*, int64_t, int, const float*, int64_t,
                     int64_t, float*, int64_t, cudaStream_t) {
    return (int)cudaErrorNotSupported;
}
}  // namespace sdb
