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
// dx_t = dS[row(t)] + sum_j dl_tj Wg[h, j]; dl_tj = dp_t p_t (delta_{j e*} - s_tj).
// Same structure as the forward gate (route.cu): a warp owns TPW tokens, lane l
// covers h = 256 i + 8 l + [0, 8), Wg from shared memory reused TPW times.
template <int EMAX, int TPW, int GW>
__global__ void __launch_bounds__(GW * 32, 1)
    gate_bwd_dx_kernel(const bf16* __restrict__ dS, const float* __restrict__ wg,
                       const float* __restrict__ logits, const int32_t* __restrict__ expert,
                       const int32_t* __restrict__ slot, const float* __restrict__ prob,
                       const float* __restrict__ dp, SlotSpace ss, int64_t T, int hch,
                       bf16* __restrict__ dx, float* __restrict__ dl_out) {
  extern __shared__ __align__(16) float ws[];  // [EMAX][hch], see ws_index
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = ss.E, H = ss.H;
  constexpr int PER_CTA = GW * TPW;
  const int nchunks = (H + hch - 1) / hch;
  const bool resident = nchunks == 1;
  if (resident) {
    stage_wg(ws, wg, 0, hch, H, E);
    __syncthreads();
  }
  const int64_t nbatch = (T + PER_CTA - 1) / PER_CTA;
  for (int64_t b = blockIdx.x; b < nbatch; b += gridDim.x) {
    const int64_t tok0 = b * PER_CTA + warp * TPW;
    float dl[TPW][EMAX];
    size_t row[TPW];
    bool kept[TPW], valid[TPW];
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int64_t tok = tok0 + t;
      valid[t] = tok < T;
      kept[t] = valid[t] && slot[tok] >= 0;
      row[t] = 0;
#pragma unroll
      for (int j = 0; j < EMAX; ++j) dl[t][j] = 0.f;
      if (kept[t]) {
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
        for (int j = 0; j < EMAX; ++j)
          dl[t][j] = j < E ? g * ((j == e ? 1.f : 0.f) - dl[t][j] * inv) : 0.f;
      }
      if (valid[t] && lane < E) {
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j == lane) v = dl[t][j];
        dl_out[(size_t)tok * E + lane] = v;
      }
      if (EMAX > 32 && valid[t] && lane + 32 < E) {
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j == lane + 32) v = dl[t][j];
        dl_out[(size_t)tok * E + lane + 32] = v;
      }
    }
    for (int c = 0; c < nchunks; ++c) {
      const int h0 = c * hch;
      if (!resident) {
        __syncthreads();
        stage_wg(ws, wg, h0, hch, H, E);
        __syncthreads();
      }
      const int hlen = H - h0 < hch ? H - h0 : hch;
      const int nblk = (hlen + 255) >> 8;
      auto load = [&](int blk, int t) -> uint4 {
        const int h = 256 * blk + 8 * lane;
        return (blk < nblk && h < hlen && kept[t]) ? ld_nc_v4(dS + row[t] + h0 + h)
                                                   : make_uint4(0, 0, 0, 0);
      };
      uint4 nxt[TPW];
#pragma unroll
      for (int t = 0; t < TPW; ++t) nxt[t] = load(0, t);
      for (int blk = 0; blk < nblk; ++blk) {
        float o[TPW][8];
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const float2 f0 = unpack_bf16x2(nxt[t].x), f1 = unpack_bf16x2(nxt[t].y);
          const float2 f2 = unpack_bf16x2(nxt[t].z), f3 = unpack_bf16x2(nxt[t].w);
          o[t][0] = f0.x; o[t][1] = f0.y; o[t][2] = f1.x; o[t][3] = f1.y;
          o[t][4] = f2.x; o[t][5] = f2.y; o[t][6] = f3.x; o[t][7] = f3.y;
        }
#pragma unroll
        for (int t = 0; t < TPW; ++t) nxt[t] = load(blk + 1, t);
        const float* wrow = ws + blk * 256 + lane * 4;
#pragma unroll
        for (int j = 0; j < EMAX; ++j) {
          const float4 w0 = *reinterpret_cast<const float4*>(wrow + j * hch);
          const float4 w1 = *reinterpret_cast<const float4*>(wrow + j * hch + 128);
#pragma unroll
          for (int t = 0; t < TPW; ++t) {
            const float d = dl[t][j];
            o[t][0] = fmaf(d, w0.x, o[t][0]); o[t][1] = fmaf(d, w0.y, o[t][1]);
            o[t][2] = fmaf(d, w0.z, o[t][2]); o[t][3] = fmaf(d, w0.w, o[t][3]);
            o[t][4] = fmaf(d, w1.x, o[t][4]); o[t][5] = fmaf(d, w1.y, o[t][5]);
            o[t][6] = fmaf(d, w1.z, o[t][6]); o[t][7] = fmaf(d, w1.w, o[t][7]);
          }
        }
        const int h = h0 + 256 * blk + 8 * lane;
        if (h - h0 < hlen) {
#pragma unroll
          for (int t = 0; t < TPW; ++t) {
            if (!valid[t]) continue;
            const uint4 v = kept[t] ? make_uint4(pack_bf16x2(o[t][0], o[t][1]), pack_bf16x2(o[t][2], o[t][3]),
                                                 pack_bf16x2(o[t][4], o[t][5]), pack_bf16x2(o[t][6], o[t][7]))
                                    : make_uint4(0, 0, 0, 0);
            st_v4(dx + (size_t)(tok0 + t) * H + h, v);
          }
        }
      }
    }
  }
}

// dWg partials: CTA = (256-wide h block, token split). Warp w handles JW experts
// (group w % NJG) over token sub-range w / NJG; lane l owns h = hb + 8 l + [0, 8).
// Per token: one 16-byte x vector and one JW-float dl vector (warp-uniform, L1),
// JW*8 FMAs as fma.rn.f32x2 over h pairs. Loads run PD tokens ahead. Sub-range
// partials are combined in shared memory in a fixed order (deterministic).
constexpr int DWG_WARPS = 8;
template <int EMAX>
__global__ void __launch_bounds__(DWG_WARPS * 32)
    dwg_partial_kernel(const bf16* __restrict__ x, const float* __restrict__ dl, int64_t T, int H,
                       int E, int64_t tok_per_split, float* __restrict__ partial) {
  constexpr int JW = EMAX <= 32 ? 4 : 8;
  constexpr int NJG = EMAX / JW > DWG_WARPS ? DWG_WARPS : EMAX / JW;
  constexpr int TSUB = DWG_WARPS / NJG;
  constexpr int PD = 4;
  __shared__ float red[DWG_WARPS][256 * JW];  // per-warp partial tiles (only when TSUB > 1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jg = warp % NJG, ts = warp / NJG;
  const int hb = blockIdx.x * 256;
  const int h = hb + 8 * lane;
  const bool hok = h < H;
  const int64_t t_begin = (int64_t)blockIdx.y * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > T) t_end = T;
  const int64_t span = (t_end - t_begin + TSUB - 1) / TSUB;
  const int64_t a0 = t_begin + ts * span;
  int64_t a1 = a0 + span;
  if (a1 > t_end) a1 = t_end;
  float2 acc[4][JW];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < JW; ++j) acc[k][j] = make_float2(0.f, 0.f);
  for (int jp = 0; jp < (EMAX / JW + NJG - 1) / NJG; ++jp) {
    const int j0 = (jg + jp * NJG) * JW;
    uint4 xb[PD];
    float db[PD][JW];
    auto load = [&](int64_t t, int slot_) {
      const bool ok = t < a1;
      xb[slot_] = (ok && hok) ? ld_nc_v4(x + (size_t)t * H + h) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < JW; ++j)
        db[slot_][j] = (ok && j0 + j < E) ? __ldg(dl + (size_t)t * E + j0 + j) : 0.f;
    };
#pragma unroll
    for (int s2 = 0; s2 < PD; ++s2) load(a0 + s2, s2);
    for (int64_t t = a0; t < a1; t += PD) {
#pragma unroll
      for (int s2 = 0; s2 < PD; ++s2) {
        if (t + s2 < a1) {
          const float2 x0 = unpack_bf16x2(xb[s2].x), x1 = unpack_bf16x2(xb[s2].y);
          const float2 x2 = unpack_bf16x2(xb[s2].z), x3 = unpack_bf16x2(xb[s2].w);
          float d[JW];
#pragma unroll
          for (int j = 0; j < JW; ++j) d[j] = db[s2][j];
          load(t + s2 + PD, s2);
#pragma unroll
          for (int j = 0; j < JW; ++j) {
            const float2 dd = make_float2(d[j], d[j]);
            ffma2(acc[0][j], x0, dd);
            ffma2(acc[1][j], x1, dd);
            ffma2(acc[2][j], x2, dd);
            ffma2(acc[3][j], x3, dd);
          }
        }
      }
    }
    // combine the TSUB token sub-ranges of this expert group (fixed order) and store
    if (TSUB > 1) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < JW; ++j) {
          red[warp][(8 * lane + 2 * k) * JW + j] = acc[k][j].x;
          red[warp][(8 * lane + 2 * k + 1) * JW + j] = acc[k][j].y;
        }
      __syncthreads();
      if (ts == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < JW; ++j) {
            float sx = 0.f, sy = 0.f;
            for (int u = 0; u < TSUB; ++u) {
              sx += red[jg + u * NJG][(8 * lane + 2 * k) * JW + j];
              sy += red[jg + u * NJG][(8 * lane + 2 * k + 1) * JW + j];
            }
            acc[k][j] = make_float2(sx, sy);
          }
      }
    }
    if (ts == 0 && hok) {
#pragma unroll
      for (int j = 0; j < JW; ++j) {
        if (j0 + j >= E) continue;
        float* dst = partial + ((size_t)blockIdx.y * H + h) * E + j0 + j;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          dst[(size_t)(2 * k) * E] = acc[k][j].x;
          dst[(size_t)(2 * k + 1) * E] = acc[k][j].y;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < JW; ++j) acc[k][j] = make_float2(0.f, 0.f);
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

int g_sms = 0;

template <int EMAX, int TPW, int GW>
cudaError_t launch_gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                            const int32_t* expert, const int32_t* slot, const float* prob,
                            const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                            float* dl, float* partial, int nsplit, cudaStream_t s) {
  constexpr int hmax = wg_chunk(EMAX);
  const int hpad = (ss.H + 255) & ~255;
  const int hch = hpad < hmax ? hpad : hmax;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_bwd_dx_kernel<EMAX, TPW, GW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t per_cta = (int64_t)GW * TPW;
  int64_t grid = (T + per_cta - 1) / per_cta;
  if (hch >= ss.H && grid > g_sms) grid = g_sms;
  gate_bwd_dx_kernel<EMAX, TPW, GW><<<(unsigned)grid, GW * 32, EMAX * hch * 4, s>>>(
      static_cast<const bf16*>(dS), wg, logits, expert, slot, prob, dp, ss, T, hch,
      static_cast<bf16*>(dx), dl);
  constexpr int EM = EMAX < 4 ? 4 : EMAX;
  const int64_t tps = (T + nsplit - 1) / nsplit;
  dim3 g2((ss.H + 255) / 256, nsplit);
  dwg_partial_kernel<EM><<<g2, DWG_WARPS * 32, 0, s>>>(static_cast<const bf16*>(x), dl, T, ss.H,
                                                       ss.E, tps, partial);
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
#define GB(EM, TP, GW) \
  launch_gate_bwd<EM, TP, GW>(x, dS, wg, logits, expert, slot, prob, dp, ss, T, dx, dwg, dl_scratch, dwg_partial, nsplit, s)
  if (ss.E <= 4) return GB(4, 8, 8);
  if (ss.E <= 8) return GB(8, 8, 8);
  if (ss.E <= 16) return GB(16, 4, 8);
  if (ss.E <= 32) return GB(32, 2, 8);
  return GB(64, 1, 8);
#undef GB
}

}  // namespace moe
