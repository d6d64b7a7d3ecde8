// optim.cu — the tiled optimizer step of include/moe_optim.h.
//
// Both paths stream the five arrays once with 16-byte accesses (8 parameters per
// thread per iteration, persistent grid-stride loop over SM-count multiples):
//   * upcast_kernel + update_kernel<f32 grads>: the paper's tiled step, one
//     4*ts-byte fp32 buffer reused by every tile;
//   * update_kernel<bf16 grads>: the fused step, the upcast happens in registers.
// The arithmetic is the same binary32 sequence in both (explicit _rn intrinsics,
// so nvcc cannot contract a multiply-add), hence bit-identical results.
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int OPT_THREADS = 256;
constexpr int OPT_VEC = 8;

__device__ __forceinline__ void adamw1(float g, float& p, float& m, float& v, const AdamwScalars& s) {
  const float m2 = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.ob1, g));
  const float v2 = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(s.ob2, __fmul_rn(g, g)));
  const float p1 = __fmul_rn(p, s.decay);
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v2), s.c2s), s.eps);
  p = __fsub_rn(p1, __fmul_rn(s.step, __fdiv_rn(m2, d)));
  m = m2;
  v = v2;
}

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

template <typename G>
__device__ __forceinline__ float grad_at(const G* g, int64_t i);
template <>
__device__ __forceinline__ float grad_at<uint16_t>(const uint16_t* g, int64_t i) { return bf16_to_f32(g[i]); }
template <>
__device__ __forceinline__ float grad_at<float>(const float* g, int64_t i) { return g[i]; }

// elements [0, n) of arrays that start at a common element offset; `head` scalar
// elements first so that the vector body is 16-byte aligned for every array
// (VEC = false: every element scalar — pointers that cannot all be aligned at once)
template <typename G, bool VEC>
__global__ void __launch_bounds__(OPT_THREADS)
    update_kernel(const G* __restrict__ g, float* __restrict__ p, float* __restrict__ m,
                  float* __restrict__ v, uint16_t* __restrict__ p16, int64_t n, int head,
                  AdamwScalars s) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (!VEC) {
    for (int64_t i = tid; i < n; i += nth) {
      float pp = p[i], mm = m[i], vv = v[i];
      adamw1(grad_at(g, i), pp, mm, vv, s);
      p[i] = pp; m[i] = mm; v[i] = vv;
      if (p16) p16[i] = __bfloat16_as_ushort(__float2bfloat16_rn(pp));
    }
    return;
  }
  if (tid < head && tid < n) {
    float pp = p[tid], mm = m[tid], vv = v[tid];
    adamw1(grad_at(g, tid), pp, mm, vv, s);
    p[tid] = pp; m[tid] = mm; v[tid] = vv;
    if (p16) p16[tid] = __bfloat16_as_ushort(__float2bfloat16_rn(pp));
  }
  const int64_t body = n > head ? (n - head) / OPT_VEC : 0;
  for (int64_t k = tid; k < body; k += nth) {
    const int64_t i = head + k * OPT_VEC;
    float gv[OPT_VEC];
    if constexpr (sizeof(G) == 2) {
      const uint4 raw = ld_nc_v4(g + i);
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        gv[2 * q] = __uint_as_float(w[q] << 16);
        gv[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
      }
    } else {
      const float4 a = *reinterpret_cast<const float4*>(g + i);
      const float4 b = *reinterpret_cast<const float4*>(g + i + 4);
      gv[0] = a.x; gv[1] = a.y; gv[2] = a.z; gv[3] = a.w;
      gv[4] = b.x; gv[5] = b.y; gv[6] = b.z; gv[7] = b.w;
    }
    float4 pa = *reinterpret_cast<const float4*>(p + i), pb = *reinterpret_cast<const float4*>(p + i + 4);
    float4 ma = *reinterpret_cast<const float4*>(m + i), mb = *reinterpret_cast<const float4*>(m + i + 4);
    float4 va = *reinterpret_cast<const float4*>(v + i), vb = *reinterpret_cast<const float4*>(v + i + 4);
    float pv[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
    float mv[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
    float vv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
#pragma unroll
    for (int q = 0; q < OPT_VEC; ++q) adamw1(gv[q], pv[q], mv[q], vv[q], s);
    *reinterpret_cast<float4*>(p + i) = make_float4(pv[0], pv[1], pv[2], pv[3]);
    *reinterpret_cast<float4*>(p + i + 4) = make_float4(pv[4], pv[5], pv[6], pv[7]);
    *reinterpret_cast<float4*>(m + i) = make_float4(mv[0], mv[1], mv[2], mv[3]);
    *reinterpret_cast<float4*>(m + i + 4) = make_float4(mv[4], mv[5], mv[6], mv[7]);
    *reinterpret_cast<float4*>(v + i) = make_float4(vv[0], vv[1], vv[2], vv[3]);
    *reinterpret_cast<float4*>(v + i + 4) = make_float4(vv[4], vv[5], vv[6], vv[7]);
    if (p16) {
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = pack_bf16x2(pv[2 * q], pv[2 * q + 1]);
      st_v4(p16 + i, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
  // tail
  const int64_t t0 = head + body * OPT_VEC;
  const int64_t i = t0 + tid;
  if (i < n && tid < OPT_VEC) {
    float pp = p[i], mm = m[i], vv = v[i];
    adamw1(grad_at(g, i), pp, mm, vv, s);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (p16) p16[i] = __bfloat16_as_ushort(__float2bfloat16_rn(pp));
  }
}

// the paper's materialised 32-bit gradients of one tile
__global__ void __launch_bounds__(OPT_THREADS)
    upcast_kernel(const uint16_t* __restrict__ g, float* __restrict__ out, int64_t n) {
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth)
    out[i] = bf16_to_f32(g[i]);
}

int g_sms = 0;

unsigned grid_for(int64_t n) {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  const int64_t want = (n / OPT_VEC + OPT_THREADS - 1) / OPT_THREADS;
  const int64_t cap = (int64_t)g_sms * 8;  // 8 resident 256-thread CTAs per SM
  return (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

namespace {
bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

template <typename G>
cudaError_t launch_update(const G* g, float* p, float* m, float* v, uint16_t* p16, int64_t n,
                          const AdamwScalars& s, cudaStream_t st) {
  // head: scalar elements before p is 16-byte aligned; the vector body needs every
  // array aligned at the same element
  const int head = (int)(((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4);
  const bool vec = (reinterpret_cast<uintptr_t>(p) & 3) == 0 && al16(g + head) && al16(m + head) &&
                   al16(v + head) && (!p16 || al16(p16 + head)) && n > head;
  if (vec)
    update_kernel<G, true><<<grid_for(n), OPT_THREADS, 0, st>>>(g, p, m, v, p16, n, head, s);
  else
    update_kernel<G, false><<<grid_for(n * OPT_VEC), OPT_THREADS, 0, st>>>(g, p, m, v, p16, n, 0, s);
  return cudaGetLastError();
}
}  // namespace

cudaError_t adamw_fused(const void* grad, float* p, float* m, float* v, void* p16, int64_t n,
                        const AdamwScalars& s, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_update(static_cast<const uint16_t*>(grad), p, m, v, static_cast<uint16_t*>(p16), n, s, st);
}

cudaError_t adamw_tiled(const void* grad, float* p, float* m, float* v, void* p16, int64_t n,
                        const AdamwScalars& s, int64_t ts, float* temp, cudaStream_t st, int* launches) {
  const uint16_t* g = static_cast<const uint16_t*>(grad);
  uint16_t* q = static_cast<uint16_t*>(p16);
  for (int64_t a = 0; a < n; a += ts) {
    const int64_t k = n - a < ts ? n - a : ts;
    upcast_kernel<<<grid_for(k * OPT_VEC), OPT_THREADS, 0, st>>>(g + a, temp, k);
    // tile sizes that are multiples of 8 keep temp and the state arrays co-aligned
    // (vector path); others fall back to the scalar kernel
    cudaError_t e = launch_update<float>(temp, p + a, m + a, v + a, q ? q + a : nullptr, k, s, st);
    *launches += 2;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace moe
