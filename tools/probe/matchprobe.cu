// Throughput of __match_any_sync vs. the number of distinct values per warp
// (1..32), against a 4-ballot equivalent; cycles per warp-instruction.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_match(unsigned* out, int distinct, int iters) {
  unsigned lane = threadIdx.x & 31, acc = 0;
  unsigned v = lane % distinct;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned m = __match_any_sync(0xFFFFFFFFu, v + (acc & 0));
    acc += m;
    v = (v + 1) % distinct + (acc & 0x100000);  // keep it data-dependent but same pattern
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)((t1 - t0) / iters);
  if (acc == 7) out[1 << 20] = acc;
}
__global__ void k_ballot(unsigned* out, int distinct, int iters) {
  unsigned lane = threadIdx.x & 31, acc = 0;
  unsigned v = lane % distinct;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned peers = 0xFFFFFFFFu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      unsigned bit = (v >> b) & 1u, m = __ballot_sync(0xFFFFFFFFu, bit);
      peers &= bit ? m : ~m;
    }
    acc += peers;
    v = (v + 1) % distinct + (acc & 0x100000);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)((t1 - t0) / iters);
  if (acc == 7) out[1 << 20] = acc;
}
int main() {
  unsigned* d; cudaMalloc(&d, (1 << 20) * 4 + 4);
  unsigned h[4];
  for (int warps : {1, 16, 32}) {
    for (int distinct : {1, 2, 4, 8, 16, 32}) {
      k_match<<<148, 32 * warps>>>(d, distinct, 4096); cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      unsigned a = h[0];
      k_ballot<<<148, 32 * warps>>>(d, distinct, 4096); cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("warps/SM=%2d distinct=%2d: match.any %4u cyc/iter  8-ballot %4u cyc/iter\n", warps, distinct, a, h[0]);
    }
  }
}
