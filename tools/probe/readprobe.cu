// Speed-of-light probe: how fast can ONE launch stream-read B bytes (and
// write a tiny result) when launches are replayed back to back from a
// CUDA graph over rotating cold buffers?  Used to bound cfg1/cfg3/cfg4.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

// pdl: 0 plain launches; 1 PDL, wait before the first read; 2 PDL, read
// first and wait only before the (tiny) write — the BTK_INPUT_READY mode.
__global__ void __launch_bounds__(512) rd(const uint4* __restrict__ x, size_t nvec, float* out, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  float acc = 0.f;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t st = (size_t)gridDim.x * blockDim.x;
#pragma unroll 8
  for (; i < nvec; i += st) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(x + i));
    acc = fmaxf(acc, __uint_as_float(v.x ^ v.y ^ v.z ^ v.w));
  }
  if (pdl == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  size_t bytes = argc > 1 ? atoll(argv[1]) : 33554432;
  int iters = 200;
  int nbuf = (int)((4ull * 126 * 1048576) / bytes) + 2;
  std::vector<void*> bufs(nbuf);
  for (auto& b : bufs) { cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes); }
  float* out; cudaMalloc(&out, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 3; ++pdl)
  for (int bpsm : {1, 2, 4, 8}) {
    int grid = 148 * bpsm;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < iters; ++i) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = grid; cfg.blockDim = 512; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, rd, (const uint4*)bufs[i % nbuf], bytes / 16, out, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double us = ms * 1e3 / iters;
    printf("bytes=%zu pdl=%d grid=%d: %.2f us/launch  %.0f GB/s\n", bytes, pdl, grid, us, bytes / us / 1e3);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
