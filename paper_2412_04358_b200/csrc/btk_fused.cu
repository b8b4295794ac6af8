// Fused interleaved fast path (placeholder until the kernel lands).
#include "btk_internal.h"

namespace btk {
bool fused_supported(const Problem&) { return false; }
cudaError_t run_fused(const Problem&, void*, int64_t*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace btk
