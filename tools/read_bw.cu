// read_bw.cu — HBM read-bandwidth probe for the gate / dWg access patterns (development tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_bw tools/read_bw.cu -lcuda
// (1) LDG.128 grid-stride over a buffer; (2) warp-per-row full rows; (3) TMA boxes
// {64 cols x R rows} walked k-block-major per CTA row tile (the gate's pattern), with
// S stages in flight; (4) TMA boxes {W cols x R rows} with W = 256 (3-D view).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int rows_total, int R,
                                                    int kblocks, int box_bytes, int ntiles, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int issued = 0, done = 0;
  const int total = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * kblocks;
  auto coords = [&](int i, int& k, int& r) {
    const int t = (int)blockIdx.x + (i / kblocks) * (int)gridDim.x;
    k = i % kblocks;
    r = t * R;
  };
  uint32_t acc = 0;
  while (done < total) {
    while (issued < total && issued - done < S) {
      const int s = issued % S;
      int k, r;
      coords(issued, k, r);
      const uint32_t bar = smem_u32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(box_bytes));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(smem + (size_t)s * box_bytes)),
          "l"(&tm), "r"(k * (box_bytes / R / 2)), "r"(r), "r"(bar)
          : "memory");
      ++issued;
    }
    const int s = done % S;
    const uint32_t ph = (uint32_t)(done / S) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(&full[s])), "r"(ph));
    acc += smem[(size_t)s * box_bytes];
    ++done;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const int T = 16384, H = 2048;
  const size_t bytes = (size_t)T * H * 2;
  void* buf;
  cudaMalloc(&buf, (size_t)1 << 30);
  cudaMemset(buf, 1, (size_t)1 << 30);
  void* flush;
  cudaMalloc(&flush, (size_t)256 << 20);
  uint32_t* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn, size_t nbytes, const char* what) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemsetAsync(flush, it, (size_t)256 << 20);
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it && ms < best) best = ms;
    }
    printf("%-60s %8.2f us  %7.1f GB/s  err=%s\n", what, best * 1e3, nbytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (size_t nb : {bytes, (size_t)1 << 30}) {
    for (int per_sm : {4, 8, 16}) {
      char w[128];
      snprintf(w, sizeof w, "LDG.128 grid-stride %zu MiB, %d x 256 thr/SM", nb >> 20, per_sm);
      timeit([&] { ldg_kernel<<<sms * per_sm, 256>>>((const uint4*)buf, nb / 16, out); }, nb, w);
    }
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int boxw : {64, 128, 256}) {
    for (int R : {112, 128, 64, 32, 16}) {
      for (int S : {4, 8}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)T};
        cuuint64_t strides[1] = {(cuuint64_t)H * 2};
        cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)R};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         boxw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int box_bytes = boxw * R * 2;
        if ((size_t)S * box_bytes + 1024 > 200 * 1024) continue;
        const int ntiles = (T + R - 1) / R;
        const int kblocks = H / boxw;
        const int smem = S * box_bytes + 1024;
        char w[128];
        snprintf(w, sizeof w, "TMA box %3d cols x %3d rows, %d stages (%d KiB in flight/SM)", boxw, R, S,
                 S * box_bytes / 1024);
        if (S == 4) {
          cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          timeit([&] { tma_kernel<4><<<ntiles < sms ? ntiles : sms, 64, smem>>>(tm, T, R, kblocks, box_bytes, ntiles, out); },
                 bytes, w);
        } else {
          cudaFuncSetAttribute(tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          timeit([&] { tma_kernel<8><<<ntiles < sms ? ntiles : sms, 64, smem>>>(tm, T, R, kblocks, box_bytes, ntiles, out); },
                 bytes, w);
        }
      }
    }
  }
  return 0;
}
