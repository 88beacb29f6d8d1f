// gemm_tc.cu -- design (b): unpack to int8 + tcgen05.mma.kind::i8 (placeholder
// until the tcgen05 kernels land; the dispatcher falls back to design (a)).
#include "bwta_internal.h"

namespace bwta {
size_t matmul_tc_workspace(const MatmulArgs&) { return 0; }
bool matmul_tc_supported(const MatmulArgs&) { return false; }
cudaError_t launch_matmul_tc(const MatmulArgs&, void*, size_t, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace bwta
