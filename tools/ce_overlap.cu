// Do peer cudaMemcpyAsync copies (copy engines) overlap a long SM-saturating kernel?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(float* out, int iters) {
  float a = threadIdx.x;
  for (int i = 0; i < iters; ++i) a = a * 1.0000001f + 0.5f;
  if (a == 12345.f) out[0] = a;
}
int main() {
  const size_t piece = 4ull << 20; const int npieces = 16;
  void *src, *dst1;
  cudaSetDevice(1); cudaMalloc(&dst1, piece * npieces);
  cudaSetDevice(0); cudaMalloc(&src, piece * npieces); cudaDeviceEnablePeerAccess(1, 0);
  float* out; cudaMalloc(&out, 4);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto copies = [&](cudaStream_t s) { for (int i = 0; i < npieces; ++i) cudaMemcpyAsync((char*)dst1 + i * piece, (char*)src + i * piece, piece, cudaMemcpyDeviceToDevice, s); };
  auto timeit = [&](auto f) { f(); cudaDeviceSynchronize(); cudaEventRecord(a); f(); cudaEventRecord(b); cudaDeviceSynchronize(); float ms; cudaEventElapsedTime(&ms, a, b); return ms; };
  int iters = 200000;
  float tk = timeit([&] { spin<<<148 * 4, 512, 0, s1>>>(out, iters); cudaStreamSynchronize(s1); });
  float tc = timeit([&] { copies(s2); cudaStreamSynchronize(s2); });
  float tb = timeit([&] { spin<<<148 * 4, 512, 0, s1>>>(out, iters); copies(s2); cudaStreamSynchronize(s1); cudaStreamSynchronize(s2); });
  printf("kernel %.3f ms, 16x4MB peer memcpy %.3f ms (%.0f GB/s), both concurrently %.3f ms\n", tk, tc, 64.0 * 1.048576 / tc, tb);
  return 0;
}
