// mc_probe.cu — is NVLink SHARP multicast (multimem) usable on this box? One process,
// two GPUs: create a multicast object over both, bind one physical allocation per GPU,
// store through the multicast address from GPU 0 and read both copies back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("%s failed: %s\n", #x, s); return 1; } } while (0)

__global__ void mc_store(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n / 4) {
    float4 v = make_float4(i, i + 0.25f, i + 0.5f, i + 0.75f);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
  }
}

int main() {
  CK(cuInit(0));
  int n = 0;
  cudaGetDeviceCount(&n);
  printf("devices %d\n", n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("dev %d multicast %d fabric_handles %d\n", d, mc, fab);
  }
  if (n < 2) return 0;
  const size_t want = 32 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 2;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = want;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (want + gran - 1) / gran * gran;
  printf("multicast granularity %zu size %zu\n", gran, mp.size);
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &mp));
  CUdevice devs[2];
  for (int d = 0; d < 2; ++d) { CK(cuDeviceGet(&devs[d], d)); CK(cuMulticastAddDevice(mch, devs[d])); }
  CUmemGenericAllocationHandle ph[2];
  CUdeviceptr ua[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMemCreate(&ph[d], mp.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph[d], 0, mp.size, 0));
    CK(cuMemAddressReserve(&ua[d], mp.size, 0, 0, 0));
    CK(cuMemMap(ua[d], mp.size, 0, ph[d], 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(ua[d], mp.size, &ad, 1));
    cudaMemset((void*)ua[d], 0, mp.size);
  }
  cudaSetDevice(0);
  CUdeviceptr mca;
  CK(cuMemAddressReserve(&mca, mp.size, 0, 0, 0));
  CK(cuMemMap(mca, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mca, mp.size, &ad, 1));
  const int nf = (int)(want / 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mc_store<<<(nf / 4 + 255) / 256, 256>>>((float*)mca, nf);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) mc_store<<<(nf / 4 + 255) / 256, 256>>>((float*)mca, nf);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("multimem.st: %s, %.1f GB/s written per destination (%.2f us per 32 MiB)\n",
         cudaGetErrorString(cudaGetLastError()), want * 10 / (ms * 1e-3) / 1e9, ms * 100);
  for (int d = 0; d < 2; ++d) {
    float h[8];
    cudaSetDevice(d);
    cudaMemcpy(h, (void*)(ua[d] + 4 * 4 * 1000), sizeof h, cudaMemcpyDeviceToHost);
    printf("dev %d copy: %.2f %.2f %.2f %.2f (want 1000.00 1000.25 1000.50 1000.75)\n", d, h[0], h[1], h[2], h[3]);
  }
  return 0;
}
