// F32 instantiation of the fused kernels (see btk_fused_impl.cuh).
#include "btk_fused_impl.cuh"

namespace btk {
namespace fz {
template cudaError_t launch_kb<F32>(const Plan&, int64_t, cudaStream_t);
}  // namespace fz
}  // namespace btk

// Development timeline trace of the fp32 kernels (each translation unit has
// its own g_trace; tools/trace_narrow.py traces fp32 configs).
extern "C" int btk_trace_read(void* host_dst, int nblocks) {
  if (nblocks > 8192) nblocks = 8192;
  return (int)cudaMemcpyFromSymbol(host_dst, btk::g_trace, (size_t)nblocks * 8 * 8);
}
