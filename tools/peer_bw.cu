// Peer NVLink bandwidth: kernel on dev 0 pushing (remote stores) into dev 1 memory vs
// pulling (remote loads) from it; plus cudaMemcpyPeerAsync. nvcc -arch=sm_100a tools/peer_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy16(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    uint4 a = s[i], b = s[i + st], c = s[i + 2 * st], e = s[i + 3 * st];
    d[i] = a; d[i + st] = b; d[i + 2 * st] = c; d[i + 3 * st] = e;
  }
  for (; i < n; i += st) d[i] = s[i];
}
int main() {
  const size_t bytes = 64ull << 20, n = bytes / 16;
  void *a0, *b0, *a1;
  cudaSetDevice(1); cudaMalloc(&a1, bytes); cudaMemset(a1, 1, bytes);
  cudaSetDevice(0); cudaMalloc(&a0, bytes); cudaMalloc(&b0, bytes); cudaMemset(a0, 1, bytes);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {148, 296, 592, 1184, 2368}) {
    for (int mode = 0; mode < 3; ++mode) {
      const uint4* s = (const uint4*)(mode == 1 ? a1 : a0);   // 0 push (local -> remote), 1 pull, 2 local
      uint4* d = (uint4*)(mode == 0 ? a1 : b0);
      copy16<<<grid, 512>>>(s, d, n);
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) copy16<<<grid, 512>>>(s, d, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %5d %-5s %7.1f GB/s\n", grid, mode == 0 ? "push" : mode == 1 ? "pull" : "local",
             bytes * 10 / (ms * 1e6));
    }
  }
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("memcpyPeer push %7.1f GB/s\n", bytes * 10 / (ms * 1e6));
  return 0;
}
