// permute.cu — the HBM-bound steps of the hot path:
//   F3  dispatch      slot-parallel gather x -> capacity-padded slot space
//   F11 combine       token-parallel y_t = p_t * O[row(t)]
//   B1  combine_bwd   dp_t = <dy_t, O[row(t)]>, dO[row(t)] = p_t dy_t
//   B10 gate_bwd      dx_t = dS[row(t)] + dl_t Wg^T, dWg = x^T dl (deterministic)
// Slot space is [G_t][E][C_s][H]: slot c of expert e lives in slice c / C_s at
// row c % C_s, so a DTD rank touches only its own slice.
// Rows move as 16-byte vectors, one warp per row/token, all loads of a row
// issued before its stores.
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int WARPS = 8;

__device__ __forceinline__ size_t slot_row(const SlotSpace& ss, int e, int64_t c) {
  const int64_t tt = c / ss.Cs, cs = c - tt * ss.Cs;
  return ((size_t)(tt * ss.E + e) * ss.Cs + cs) * ss.H;
}

// Copies one H-row (nv 16-byte vectors) with U vectors in flight per lane.
template <bool ZERO>
__device__ __forceinline__ void copy_row(const bf16* __restrict__ src, bf16* __restrict__ dst,
                                         int nv, int lane) {
  constexpr int U = 8;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    uint4 buf[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      buf[u] = (!ZERO && v < nv) ? ld_nc_v4(src + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) st_v4(dst + (size_t)v * 8, buf[u]);
    }
  }
}

__global__ void __launch_bounds__(WARPS * 32)
    dispatch_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ tok_of,
                    const int32_t* __restrict__ count, SlotSpace ss, int t_lo, int64_t rows,
                    bf16* __restrict__ D) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t per_slice = (int64_t)ss.E * ss.Cs;
  const int tt = t_lo + (int)(r / per_slice);
  const int64_t rem = r % per_slice;
  const int e = (int)(rem / ss.Cs);
  const int64_t cs = rem % ss.Cs;
  const int64_t c = (int64_t)tt * ss.Cs + cs;
  bf16* dst = D + ((size_t)(tt * ss.E + e) * ss.Cs + cs) * ss.H;
  const int nv = ss.H / 8;
  if (c < count[e]) {
    const int t = tok_of[(size_t)e * ss.C + c];
    copy_row<false>(x + (size_t)t * ss.H, dst, nv, lane);
  } else {
    copy_row<true>(nullptr, dst, nv, lane);
  }
}

__global__ void __launch_bounds__(WARPS * 32)
    combine_kernel(const bf16* __restrict__ O, const int32_t* __restrict__ expert,
                   const int32_t* __restrict__ slot, const float* __restrict__ prob, SlotSpace ss,
                   int64_t T, bf16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= T) return;
  const int s = slot[t];
  const int nv = ss.H / 8;
  bf16* dst = y + (size_t)t * ss.H;
  if (s < 0) {
    copy_row<true>(nullptr, dst, nv, lane);
    return;
  }
  const bf16* src = O + slot_row(ss, expert[t], s);
  const float p = prob[t];
  constexpr int U = 8;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    uint4 buf[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      buf[u] = v < nv ? ld_nc_v4(src + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) {
        uint32_t w[4] = {buf[u].x, buf[u].y, buf[u].z, buf[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 f = unpack_bf16x2(w[k]);
          w[k] = pack_bf16x2(p * f.x, p * f.y);
        }
        st_v4(dst + (size_t)v * 8, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
  }
}

__global__ void __launch_bounds__(WARPS * 32)
    combine_bwd_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ O,
                       const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                       const float* __restrict__ prob, SlotSpace ss, int64_t T, int t_lo,
                       int t_hi, float* __restrict__ dp, bf16* __restrict__ dO) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= T) return;
  const int s = slot[t];
  if (s < 0) {
    if (lane == 0) dp[t] = 0.f;
    return;
  }
  const size_t row = slot_row(ss, expert[t], s);
  const int tt = (int)(s / ss.Cs);
  const bool mine = tt >= t_lo && tt < t_hi;
  const float p = prob[t];
  const bf16* dyr = dy + (size_t)t * ss.H;
  const bf16* orow = O + row;
  bf16* dst = dO + row;
  const int nv = ss.H / 8;
  float acc = 0.f;
  constexpr int U = 4;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      a[u] = v < nv ? ld_nc_v4(dyr + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
      b[u] = v < nv ? ld_nc_v4(orow + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      uint32_t wa[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
      uint32_t wb[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 fa = unpack_bf16x2(wa[k]), fb = unpack_bf16x2(wb[k]);
        acc = fmaf(fa.x, fb.x, acc);
        acc = fmaf(fa.y, fb.y, acc);
        w[k] = pack_bf16x2(p * fa.x, p * fa.y);
      }
      if (mine && v < nv) st_v4(dst + (size_t)v * 8, make_uint4(w[0], w[1], w[2], w[3]));
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) dp[t] = acc;
}

// zero-fill the empty slots (c >= count[e]) of slices [t_lo, t_hi)
__global__ void __launch_bounds__(WARPS * 32)
    zero_empty_kernel(const int32_t* __restrict__ count, SlotSpace ss, int t_lo, int64_t rows,
                      bf16* __restrict__ D) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t per_slice = (int64_t)ss.E * ss.Cs;
  const int tt = t_lo + (int)(r / per_slice);
  const int64_t rem = r % per_slice;
  const int e = (int)(rem / ss.Cs);
  const int64_t cs = rem % ss.Cs;
  if ((int64_t)tt * ss.Cs + cs < count[e]) return;
  copy_row<true>(nullptr, D + ((size_t)(tt * ss.E + e) * ss.Cs + cs) * ss.H, ss.H / 8, lane);
}

// ---------------------------------------------------------------- B10 gate backward
constexpr int HC = 256;

// dx_t = dS[row(t)] + sum_j dl_tj Wg[h, j]; dl_tj = dp_t p_t (delta_{j e*} - s_tj).
template <int EMAX, int TPW>
__global__ void __launch_bounds__(WARPS * 32)
    gate_bwd_dx_kernel(const bf16* __restrict__ dS, const float* __restrict__ wg,
                       const float* __restrict__ logits, const int32_t* __restrict__ expert,
                       const int32_t* __restrict__ slot, const float* __restrict__ prob,
                       const float* __restrict__ dp, SlotSpace ss, int64_t T,
                       bf16* __restrict__ dx, float* __restrict__ dl_out) {
  extern __shared__ __align__(16) float ws[];  // [EMAX * HC]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tok0 = ((int64_t)blockIdx.x * WARPS + warp) * TPW;
  const int E = ss.E, H = ss.H;
  float dl[TPW][EMAX];
  size_t row[TPW];
  bool kept[TPW];
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int64_t tok = tok0 + t;
    kept[t] = false;
    row[t] = 0;
#pragma unroll
    for (int j = 0; j < EMAX; ++j) dl[t][j] = 0.f;
    if (tok < T && slot[tok] >= 0) {
      kept[t] = true;
      const int e = expert[tok];
      row[t] = slot_row(ss, e, slot[tok]);
      float m = -3.402823e38f;
#pragma unroll
      for (int j = 0; j < EMAX; ++j)
        if (j < E) m = fmaxf(m, logits[(size_t)tok * E + j]);
      float den = 0.f;
#pragma unroll
      for (int j = 0; j < EMAX; ++j)
        if (j < E) {
          dl[t][j] = expf(logits[(size_t)tok * E + j] - m);
          den += dl[t][j];
        }
      const float g = dp[tok] * prob[tok];
      const float inv = 1.0f / den;
#pragma unroll
      for (int j = 0; j < EMAX; ++j) dl[t][j] = g * ((j == e ? 1.f : 0.f) - dl[t][j] * inv);
    }
    if (tok < T && lane < EMAX && lane < E) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < EMAX; ++j)
        if (j == lane) v = dl[t][j];
      dl_out[(size_t)tok * E + lane] = v;
      if (EMAX > 32 && lane + 32 < E) {
        float v2 = 0.f;
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j == lane + 32) v2 = dl[t][j];
        dl_out[(size_t)tok * E + lane + 32] = v2;
      }
    }
  }
  for (int h0 = 0; h0 < H; h0 += HC) {
    __syncthreads();
    for (int i = threadIdx.x; i < EMAX * HC; i += blockDim.x) {
      const int j = i / HC, hl = i % HC;
      const int l = hl >> 3, half = (hl >> 2) & 1, q = hl & 3;
      const int h = h0 + hl;
      ws[j * HC + half * 128 + l * 4 + q] = (j < E && h < H) ? wg[(size_t)h * E + j] : 0.f;
    }
    __syncthreads();
    const int h = h0 + 8 * lane;
    if (h >= H) continue;
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int64_t tok = tok0 + t;
      if (tok >= T) continue;
      bf16* dst = dx + (size_t)tok * H + h;
      if (!kept[t]) {
        st_v4(dst, make_uint4(0, 0, 0, 0));
        continue;
      }
      const uint4 u = ld_nc_v4(dS + row[t] + h);
      float o[8];
      float2 f0 = unpack_bf16x2(u.x), f1 = unpack_bf16x2(u.y), f2 = unpack_bf16x2(u.z),
             f3 = unpack_bf16x2(u.w);
      o[0] = f0.x; o[1] = f0.y; o[2] = f1.x; o[3] = f1.y;
      o[4] = f2.x; o[5] = f2.y; o[6] = f3.x; o[7] = f3.y;
      float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < EMAX; ++j) {
        const float4 w0 = *reinterpret_cast<const float4*>(&ws[j * HC + lane * 4]);
        const float4 w1 = *reinterpret_cast<const float4*>(&ws[j * HC + 128 + lane * 4]);
        const float d = dl[t][j];
        g[0] = fmaf(d, w0.x, g[0]); g[1] = fmaf(d, w0.y, g[1]);
        g[2] = fmaf(d, w0.z, g[2]); g[3] = fmaf(d, w0.w, g[3]);
        g[4] = fmaf(d, w1.x, g[4]); g[5] = fmaf(d, w1.y, g[5]);
        g[6] = fmaf(d, w1.z, g[6]); g[7] = fmaf(d, w1.w, g[7]);
      }
      st_v4(dst, make_uint4(pack_bf16x2(o[0] + g[0], o[1] + g[1]), pack_bf16x2(o[2] + g[2], o[3] + g[3]),
                            pack_bf16x2(o[4] + g[4], o[5] + g[5]), pack_bf16x2(o[6] + g[6], o[7] + g[7])));
    }
  }
}

// dWg partials: CTA (h block of 256, token split s) -> partial[s][h][j].
// Thread (hq, jg): 4 consecutive h x EMAX/4 experts.
constexpr int DWG_TT = 32;
template <int EMAX>
__global__ void __launch_bounds__(256)
    dwg_partial_kernel(const bf16* __restrict__ x, const float* __restrict__ dl, int64_t T, int H,
                       int E, int64_t tok_per_split, float* __restrict__ partial) {
  constexpr int EJ = EMAX / 4;
  __shared__ __align__(16) float xs[DWG_TT][HC];
  __shared__ __align__(16) float ds[DWG_TT][EMAX];
  const int hq = threadIdx.x & 63, jg = threadIdx.x >> 6;
  const int h0 = blockIdx.x * HC;
  const int64_t t_begin = (int64_t)blockIdx.y * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > T) t_end = T;
  float acc[4][EJ];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < EJ; ++j) acc[a][j] = 0.f;
  for (int64_t tb = t_begin; tb < t_end; tb += DWG_TT) {
    __syncthreads();
    for (int i = threadIdx.x; i < DWG_TT * (HC / 8); i += 256) {
      const int tt = i / (HC / 8), v = i % (HC / 8);
      const int64_t t = tb + tt;
      const int h = h0 + v * 8;
      float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (t < t_end && h < H) {
        const uint4 u = ld_nc_v4(x + (size_t)t * H + h);
        float2 a0 = unpack_bf16x2(u.x), a1 = unpack_bf16x2(u.y), a2 = unpack_bf16x2(u.z),
               a3 = unpack_bf16x2(u.w);
        f[0] = a0.x; f[1] = a0.y; f[2] = a1.x; f[3] = a1.y;
        f[4] = a2.x; f[5] = a2.y; f[6] = a3.x; f[7] = a3.y;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) xs[tt][v * 8 + k] = f[k];
    }
    for (int i = threadIdx.x; i < DWG_TT * EMAX; i += 256) {
      const int tt = i / EMAX, j = i % EMAX;
      const int64_t t = tb + tt;
      ds[tt][j] = (t < t_end && j < E) ? dl[(size_t)t * E + j] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int tt = 0; tt < DWG_TT; ++tt) {
      const float4 xv = *reinterpret_cast<const float4*>(&xs[tt][hq * 4]);
      float dv[EJ];
#pragma unroll
      for (int j = 0; j < EJ; ++j) dv[j] = ds[tt][jg * EJ + j];
#pragma unroll
      for (int j = 0; j < EJ; ++j) {
        acc[0][j] = fmaf(xv.x, dv[j], acc[0][j]);
        acc[1][j] = fmaf(xv.y, dv[j], acc[1][j]);
        acc[2][j] = fmaf(xv.z, dv[j], acc[2][j]);
        acc[3][j] = fmaf(xv.w, dv[j], acc[3][j]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int h = h0 + hq * 4 + a;
    if (h >= H) continue;
#pragma unroll
    for (int j = 0; j < EJ; ++j) {
      const int jj = jg * EJ + j;
      if (jj < E) partial[((size_t)blockIdx.y * H + h) * E + jj] = acc[a][j];
    }
  }
}

__global__ void dwg_reduce_kernel(const float* __restrict__ partial, int nsplit, int64_t n,
                                  float* __restrict__ dwg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int k = 0; k < nsplit; ++k) s += partial[(size_t)k * n + i];
  dwg[i] = s;
}

template <int EMAX, int TPW>
cudaError_t launch_gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                            const int32_t* expert, const int32_t* slot, const float* prob,
                            const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                            float* dl, float* partial, int nsplit, cudaStream_t s) {
  const int64_t per_cta = (int64_t)WARPS * TPW;
  const unsigned grid = (unsigned)((T + per_cta - 1) / per_cta);
  const int smem = EMAX * HC * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_bwd_dx_kernel<EMAX, TPW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gate_bwd_dx_kernel<EMAX, TPW><<<grid, WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(dS), wg, logits, expert, slot, prob, dp, ss, T,
      static_cast<bf16*>(dx), dl);
  const int64_t tps = ((T + nsplit - 1) / nsplit + DWG_TT - 1) / DWG_TT * DWG_TT;
  constexpr int EM = EMAX < 4 ? 4 : EMAX;
  dim3 g2((ss.H + HC - 1) / HC, nsplit);
  dwg_partial_kernel<EM><<<g2, 256, 0, s>>>(static_cast<const bf16*>(x), dl, T, ss.H, ss.E, tps,
                                            partial);
  const int64_t n = (int64_t)ss.H * ss.E;
  dwg_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(partial, nsplit, n, dwg);
  return cudaGetLastError();
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + WARPS - 1) / WARPS); }

}  // namespace

int gate_bwd_splits(int64_t T) {
  int64_t s = T / 512;
  if (s < 1) s = 1;
  if (s > 32) s = 32;
  return (int)s;
}

cudaError_t dispatch(const void* x, const int32_t* tok_of, const int32_t* count,
                     const SlotSpace& ss, int t_lo, int t_hi, void* D, cudaStream_t s) {
  const int64_t rows = (int64_t)(t_hi - t_lo) * ss.E * ss.Cs;
  if (rows <= 0) return cudaSuccess;
  dispatch_kernel<<<blocks_for(rows), WARPS * 32, 0, s>>>(static_cast<const bf16*>(x), tok_of,
                                                           count, ss, t_lo, rows,
                                                           static_cast<bf16*>(D));
  return cudaGetLastError();
}

cudaError_t combine(const void* O, const int32_t* expert, const int32_t* slot, const float* prob,
                    const SlotSpace& ss, int64_t T, void* y, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  combine_kernel<<<blocks_for(T), WARPS * 32, 0, s>>>(static_cast<const bf16*>(O), expert, slot,
                                                       prob, ss, T, static_cast<bf16*>(y));
  return cudaGetLastError();
}

cudaError_t combine_bwd(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                        const float* prob, const int32_t* count, const SlotSpace& ss, int64_t T,
                        int t_lo, int t_hi, float* dp, void* dO, cudaStream_t s) {
  if (T > 0)
    combine_bwd_kernel<<<blocks_for(T), WARPS * 32, 0, s>>>(
        static_cast<const bf16*>(dy), static_cast<const bf16*>(O), expert, slot, prob, ss, T, t_lo,
        t_hi, dp, static_cast<bf16*>(dO));
  const int64_t rows = (int64_t)(t_hi - t_lo) * ss.E * ss.Cs;
  if (rows > 0)
    zero_empty_kernel<<<blocks_for(rows), WARPS * 32, 0, s>>>(count, ss, t_lo, rows,
                                                               static_cast<bf16*>(dO));
  return cudaGetLastError();
}

cudaError_t gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                     const int32_t* expert, const int32_t* slot, const float* prob,
                     const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                     float* dl_scratch, float* dwg_partial, int nsplit, cudaStream_t s) {
  if (T <= 0) return cudaMemsetAsync(dwg, 0, sizeof(float) * ss.H * ss.E, s);
#define GB(EM, TP) \
  launch_gate_bwd<EM, TP>(x, dS, wg, logits, expert, slot, prob, dp, ss, T, dx, dwg, dl_scratch, dwg_partial, nsplit, s)
  if (ss.E <= 4) return GB(4, 8);
  if (ss.E <= 8) return GB(8, 8);
  if (ss.E <= 16) return GB(16, 4);
  if (ss.E <= 32) return GB(32, 2);
  return GB(64, 1);
#undef GB
}

}  // namespace moe
