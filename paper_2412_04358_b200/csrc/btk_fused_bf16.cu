// BF16 instantiation of the fused kernels (see btk_fused_impl.cuh).
#include "btk_fused_impl.cuh"

namespace btk {
namespace fz {
template cudaError_t launch_kb<BF16>(const Plan&, int64_t, cudaStream_t);
}  // namespace fz
}  // namespace btk
