// common.cuh — device helpers shared by the sm_100a kernels of libmoe.
// Inline PTX wrappers for mbarrier / TMA / tcgen05, bf16 packing and the
// GeLU (tanh form, reading R8) used by the GEMM epilogues.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

typedef __nv_bfloat16 bf16;

// ---------------------------------------------------------------- scalar math
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// gelu_tanh(h) = 0.5 h (1 + tanh(sqrt(2/pi) (h + 0.044715 h^3)))
__device__ __forceinline__ float gelu_f(float h) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * h, h * h, h);
  return 0.5f * h * (1.0f + tanh_fast(u));
}

// d gelu_tanh / dh
__device__ __forceinline__ float gelu_grad_f(float h) {
  const float k = 0.7978845608028654f;
  const float u = k * fmaf(0.044715f * h, h * h, h);
  const float th = tanh_fast(u);
  return 0.5f * (1.0f + th) + 0.5f * h * (1.0f - th * th) * k * fmaf(3.0f * 0.044715f, h * h, 1.0f);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
  float2 r;
  r.x = __uint_as_float(u << 16);
  r.y = __uint_as_float(u & 0xFFFF0000u);
  return r;
}

// ---------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* desc, uint32_t bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem], cta_group::1, kind::f16 (bf16 in, fp32 accumulate).
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05.mma has completed.
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- 16-byte global access
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// One 16-byte store through an NVLink SHARP multicast mapping: the switch writes it to
// every member of the multicast object (bits copied as-is).
__device__ __forceinline__ void st_mc_v4(void* p, uint4 v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace moe

namespace moe {

// ---------------------------------------------------------------- packed fp32 (sm_100)
// d.xy += a.xy * b.xy in one fma.rn.f32x2 (two IEEE fp32 FMAs).
__device__ __forceinline__ void ffma2(float2& d, const float2 a, const float2 b) {
  unsigned long long& dd = *reinterpret_cast<unsigned long long*>(&d);
  asm("fma.rn.f32x2 %0, %1, %2, %0;"
      : "+l"(dd)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
}

// Largest multiple of 256 with hch * emax * 4 <= 128 KiB.
__host__ __device__ constexpr int wg_chunk(int emax) { return (128 * 1024 / (emax * 4)) & ~255; }

}  // namespace moe

namespace moe {

// ---------------------------------------------------------------- clusters / CTA pairs
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive on the mbarrier at the same shared-memory offset in CTA `cta` of the cluster.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar),
      "r"(cta)
      : "memory");
}

// 2-SM TMA load: data lands in this CTA's shared memory, transaction bytes are
// counted on the pair leader's mbarrier (peer bit cleared, as CUTLASS does).
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const void* desc, uint32_t bar, int c0,
                                                int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// D[tmem] (+)= A . B over the CTA pair (M = 256), issued by the leader CTA only.
__device__ __forceinline__ void tc_mma_f16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Commit the pair's outstanding MMAs to the mbarrier at `bar` in every CTA of `mask`.
__device__ __forceinline__ void tc_commit_2sm(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"(mask)
      : "memory");
}

}  // namespace moe

namespace moe {

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

}  // namespace moe

namespace moe {

// ---------------------------------------------------------------- legacy warp MMA (small GEMMs)
// D(16x8, fp32) += A(16x16, bf16, row) . B(16x8, bf16, col): used only for the
// gate-gradient contractions (K = E or N = E), where the fp32 operand is split
// into bf16 hi + lo and the 1e-2 gradient tolerance applies.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// fp32 -> (hi, lo) bf16 with hi + lo == v to ~2^-17 relative.
__device__ __forceinline__ void split_bf16(float v, bf16& hi, bf16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

__device__ __forceinline__ uint32_t pack2(bf16 a, bf16 b) {
  return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}

}  // namespace moe

namespace moe {

// ---------------------------------------------------------------- cp.async (16 B)
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

}  // namespace moe

namespace moe {

// ---------------------------------------------------------------- packed fp32 epilogue math
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long u) { return *reinterpret_cast<float2*>(&u); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}

// gelu_tanh on a pair (same formula as gelu_f)
__device__ __forceinline__ float2 gelu2(float2 h) {
  const float k = 0.7978845608028654f, c = 0.044715f;
  const float2 h2 = f2mul(h, h);
  const float2 t = f2fma(h2, make_float2(c, c), make_float2(1.f, 1.f));  // 1 + c h^2
  const float2 u = f2mul(f2mul(h, make_float2(k, k)), t);
  const float2 th = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 hh = f2mul(h, make_float2(0.5f, 0.5f));
  return f2fma(hh, th, hh);  // 0.5 h (1 + tanh u)
}

// d gelu_tanh / dh on a pair (same formula as gelu_grad_f)
__device__ __forceinline__ float2 gelu_grad2(float2 h) {
  const float k = 0.7978845608028654f, c = 0.044715f;
  const float2 h2 = f2mul(h, h);
  const float2 t = f2fma(h2, make_float2(c, c), make_float2(1.f, 1.f));
  const float2 kh = f2mul(h, make_float2(k, k));
  const float2 u = f2mul(kh, t);
  const float2 th = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 a = f2fma(th, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));            // 0.5 (1 + th)
  const float2 s = f2fma(f2mul(th, th), make_float2(-1.f, -1.f), make_float2(1.f, 1.f));   // 1 - th^2
  const float2 b = f2fma(h2, make_float2(3.f * c, 3.f * c), make_float2(1.f, 1.f));         // 1 + 3 c h^2
  return f2fma(f2mul(f2mul(kh, make_float2(0.5f, 0.5f)), s), b, a);
}

// gelu_tanh and its derivative on a pair, sharing u and tanh(u) (same formulas as
// gelu2 / gelu_grad2: the F6 epilogue needs both)
__device__ __forceinline__ void gelu_and_grad2(float2 h, float2& g, float2& gp) {
  const float k = 0.7978845608028654f, c = 0.044715f;
  const float2 h2 = f2mul(h, h);
  const float2 t = f2fma(h2, make_float2(c, c), make_float2(1.f, 1.f));
  const float2 kh = f2mul(h, make_float2(k, k));
  const float2 u = f2mul(kh, t);
  const float2 th = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 hh = f2mul(h, make_float2(0.5f, 0.5f));
  g = f2fma(hh, th, hh);
  const float2 a = f2fma(th, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
  const float2 s = f2fma(f2mul(th, th), make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
  const float2 b = f2fma(h2, make_float2(3.f * c, 3.f * c), make_float2(1.f, 1.f));
  gp = f2fma(f2mul(f2mul(kh, make_float2(0.5f, 0.5f)), s), b, a);
}

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr)
               : "memory");
  return r;
}

}  // namespace moe
