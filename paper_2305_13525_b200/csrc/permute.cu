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
constexpr int PD = 4;  // prefetch depth (64-wide H steps) of the gate-backward pipeline

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
// Same lane layout and Wg staging as the forward gate (route.cu): 4 token groups
// of 8 lanes per warp, TPW tokens per lane, packed fma.rn.f32x2 over h pairs.
template <int EMAX, int TPW, int GW>
__global__ void __launch_bounds__(GW * 32, 1)
    gate_bwd_dx_kernel(const bf16* __restrict__ dS, const float* __restrict__ wg,
                       const float* __restrict__ logits, const int32_t* __restrict__ expert,
                       const int32_t* __restrict__ slot, const float* __restrict__ prob,
                       const float* __restrict__ dp, SlotSpace ss, int64_t T, int hch,
                       bf16* __restrict__ dx, float* __restrict__ dl_out) {
  extern __shared__ __align__(16) float ws[];  // [EMAX][hch], see ws_index
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane >> 3, l8 = lane & 7;
  const int E = ss.E, H = ss.H;
  constexpr int PER_WARP = 4 * TPW;
  constexpr int PER_CTA = GW * PER_WARP;
  const int nchunks = (H + hch - 1) / hch;
  const bool resident = nchunks == 1;
  if (resident) {
    stage_wg(ws, wg, 0, hch, H, E);
    __syncthreads();
  }
  const int64_t nbatch = (T + PER_CTA - 1) / PER_CTA;
  for (int64_t b = blockIdx.x; b < nbatch; b += gridDim.x) {
    const int64_t base = b * PER_CTA + warp * PER_WARP + q;
    float2 dl2[TPW][EMAX];  // (dl, dl) pairs
    size_t row[TPW];
    bool kept[TPW], valid[TPW];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t tok = base + 4 * i;
      valid[i] = tok < T;
      kept[i] = valid[i] && slot[tok] >= 0;
      row[i] = 0;
      float d[EMAX];
#pragma unroll
      for (int j = 0; j < EMAX; ++j) d[j] = 0.f;
      if (kept[i]) {
        const int e = expert[tok];
        row[i] = slot_row(ss, e, slot[tok]);
        float m = -3.402823e38f;
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j < E) m = fmaxf(m, logits[(size_t)tok * E + j]);
        float den = 0.f;
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j < E) {
            d[j] = expf(logits[(size_t)tok * E + j] - m);
            den += d[j];
          }
        const float g = dp[tok] * prob[tok];
        const float inv = 1.0f / den;
#pragma unroll
        for (int j = 0; j < EMAX; ++j) d[j] = j < E ? g * ((j == e ? 1.f : 0.f) - d[j] * inv) : 0.f;
      }
      if (valid[i] && l8 == 0) {
#pragma unroll
        for (int j = 0; j < EMAX; ++j)
          if (j < E) dl_out[(size_t)tok * E + j] = d[j];
      }
#pragma unroll
      for (int j = 0; j < EMAX; ++j) dl2[i][j] = make_float2(d[j], d[j]);
    }
    for (int c = 0; c < nchunks; ++c) {
      const int h0 = c * hch;
      if (!resident) {
        __syncthreads();
        stage_wg(ws, wg, h0, hch, H, E);
        __syncthreads();
      }
      const int nblk = (H - h0 < hch ? H - h0 : hch) >> 6;
      // software pipeline: dS for steps blk .. blk+PD-1 in flight
      uint4 buf[PD][TPW];
#pragma unroll
      for (int s = 0; s < PD; ++s)
#pragma unroll
        for (int i = 0; i < TPW; ++i)
          buf[s][i] = (kept[i] && s < nblk) ? ld_nc_v4(dS + row[i] + h0 + 64 * s + 8 * l8)
                                            : make_uint4(0, 0, 0, 0);
      for (int blk0 = 0; blk0 < nblk; blk0 += PD) {
#pragma unroll
        for (int s = 0; s < PD; ++s) {
          const int blk = blk0 + s;
          if (blk < nblk) {
            const int h = h0 + 64 * blk + 8 * l8;
            float2 o[TPW][4];
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
              o[i][0] = unpack_bf16x2(buf[s][i].x); o[i][1] = unpack_bf16x2(buf[s][i].y);
              o[i][2] = unpack_bf16x2(buf[s][i].z); o[i][3] = unpack_bf16x2(buf[s][i].w);
              if (kept[i] && blk + PD < nblk) buf[s][i] = ld_nc_v4(dS + row[i] + h + 64 * PD);
            }
            const float* wrow = ws + blk * 64 + l8 * 4;
#pragma unroll
            for (int j = 0; j < EMAX; ++j) {
              const float4 w0 = *reinterpret_cast<const float4*>(wrow + j * hch);
              const float4 w1 = *reinterpret_cast<const float4*>(wrow + j * hch + 32);
              const float2 p0 = make_float2(w0.x, w0.y), p1 = make_float2(w0.z, w0.w);
              const float2 p2 = make_float2(w1.x, w1.y), p3 = make_float2(w1.z, w1.w);
#pragma unroll
              for (int i = 0; i < TPW; ++i) {
                ffma2(o[i][0], dl2[i][j], p0);
                ffma2(o[i][1], dl2[i][j], p1);
                ffma2(o[i][2], dl2[i][j], p2);
                ffma2(o[i][3], dl2[i][j], p3);
              }
            }
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
              if (!valid[i]) continue;
              const uint4 v = kept[i] ? make_uint4(pack_bf16x2(o[i][0].x, o[i][0].y),
                                                   pack_bf16x2(o[i][1].x, o[i][1].y),
                                                   pack_bf16x2(o[i][2].x, o[i][2].y),
                                                   pack_bf16x2(o[i][3].x, o[i][3].y))
                                      : make_uint4(0, 0, 0, 0);
              st_v4(dx + (size_t)(base + 4 * i) * H + h, v);
            }
          }
        }
      }
    }
  }
}

// dWg = x^T dl: CTA (h block of HB, token split) -> partial[split][h][j]. Thread
// tile 8 h x JT j; x tile staged as fp32 [TT][half][hq][4] (conflict-free LDS.128),
// dl staged as (dl, dl) pairs so fma.rn.f32x2 runs over h pairs.
constexpr int DWG_TT = 16;
template <int EMAX>
__global__ void __launch_bounds__(256, 1)
    dwg_partial_kernel(const bf16* __restrict__ x, const float* __restrict__ dl, int64_t T, int H,
                       int E, int64_t tok_per_split, float* __restrict__ partial) {
  constexpr int JT = EMAX < 8 ? EMAX : 8;
  constexpr int JG = EMAX / JT;
  constexpr int HQ = (256 / JG) < 64 ? (256 / JG) : 64;  // threads along h
  constexpr int NT = HQ * JG;                              // threads per CTA
  constexpr int HB = HQ * 8;                               // h per CTA
  __shared__ __align__(16) float xs[DWG_TT][HB];
  __shared__ __align__(16) float2 ds[DWG_TT][EMAX];
  const int hq = threadIdx.x % HQ, jg = threadIdx.x / HQ;
  const int hbase = blockIdx.x * HB;
  const int64_t t_begin = (int64_t)blockIdx.y * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > T) t_end = T;
  float2 acc[4][JT];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < JT; ++j) acc[a][j] = make_float2(0.f, 0.f);
  // register-staged double buffering: the next tile's x / dl loads are in flight
  // while the current tile is consumed from shared memory
  constexpr int XV = (DWG_TT * HQ + NT - 1) / NT;
  constexpr int DV = (DWG_TT * EMAX + NT - 1) / NT;
  uint4 xr[XV];
  float dr[DV];
  auto load_tile = [&](int64_t tb) {
#pragma unroll
    for (int k = 0; k < XV; ++k) {
      const int i = threadIdx.x + k * NT;
      const int tt = i / HQ, v = i % HQ;
      const int64_t t = tb + tt;
      const int h = hbase + v * 8;
      xr[k] = (i < DWG_TT * HQ && t < t_end && h < H) ? ld_nc_v4(x + (size_t)t * H + h)
                                                        : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < DV; ++k) {
      const int i = threadIdx.x + k * NT;
      const int tt = i / EMAX, j = i % EMAX;
      const int64_t t = tb + tt;
      dr[k] = (i < DWG_TT * EMAX && t < t_end && j < E) ? dl[(size_t)t * E + j] : 0.f;
    }
  };
  if (t_begin < t_end) load_tile(t_begin);
  for (int64_t tb = t_begin; tb < t_end; tb += DWG_TT) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < XV; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i >= DWG_TT * HQ) continue;
      const int tt = i / HQ, v = i % HQ;
      const float2 a0 = unpack_bf16x2(xr[k].x), a1 = unpack_bf16x2(xr[k].y),
                   a2 = unpack_bf16x2(xr[k].z), a3 = unpack_bf16x2(xr[k].w);
      *reinterpret_cast<float4*>(&xs[tt][v * 4]) = make_float4(a0.x, a0.y, a1.x, a1.y);
      *reinterpret_cast<float4*>(&xs[tt][HB / 2 + v * 4]) = make_float4(a2.x, a2.y, a3.x, a3.y);
    }
#pragma unroll
    for (int k = 0; k < DV; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < DWG_TT * EMAX) ds[i / EMAX][i % EMAX] = make_float2(dr[k], dr[k]);
    }
    __syncthreads();
    if (tb + DWG_TT < t_end) load_tile(tb + DWG_TT);
#pragma unroll 2
    for (int tt = 0; tt < DWG_TT; ++tt) {
      const float4 xa = *reinterpret_cast<const float4*>(&xs[tt][hq * 4]);
      const float4 xb = *reinterpret_cast<const float4*>(&xs[tt][HB / 2 + hq * 4]);
      const float2 x0 = make_float2(xa.x, xa.y), x1 = make_float2(xa.z, xa.w);
      const float2 x2 = make_float2(xb.x, xb.y), x3 = make_float2(xb.z, xb.w);
#pragma unroll
      for (int j = 0; j < JT; ++j) {
        const float2 d = ds[tt][jg * JT + j];
        ffma2(acc[0][j], x0, d);
        ffma2(acc[1][j], x1, d);
        ffma2(acc[2][j], x2, d);
        ffma2(acc[3][j], x3, d);
      }
    }
  }
  const int h = hbase + hq * 8;
  if (h >= H) return;
#pragma unroll
  for (int j = 0; j < JT; ++j) {
    const int jj = jg * JT + j;
    if (jj >= E) continue;
    float* dst = partial + ((size_t)blockIdx.y * H + h) * E + jj;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      dst[(size_t)(2 * a) * E] = acc[a][j].x;
      dst[(size_t)(2 * a + 1) * E] = acc[a][j].y;
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

int g_sms = 0;

template <int EMAX, int TPW, int GW>
cudaError_t launch_gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                            const int32_t* expert, const int32_t* slot, const float* prob,
                            const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                            float* dl, float* partial, int nsplit, cudaStream_t s) {
  constexpr int hmax = wg_chunk(EMAX);
  const int hch = ss.H < hmax ? ss.H : hmax;
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
  const int64_t per_cta = (int64_t)GW * 4 * TPW;
  int64_t grid = (T + per_cta - 1) / per_cta;
  if (hch >= ss.H && grid > g_sms) grid = g_sms;
  gate_bwd_dx_kernel<EMAX, TPW, GW><<<(unsigned)grid, GW * 32, EMAX * hch * 4, s>>>(
      static_cast<const bf16*>(dS), wg, logits, expert, slot, prob, dp, ss, T, hch,
      static_cast<bf16*>(dx), dl);
  constexpr int EM = EMAX < 4 ? 4 : EMAX;
  constexpr int JT = EM < 8 ? EM : 8;
  constexpr int HQ = (256 / (EM / JT)) < 64 ? (256 / (EM / JT)) : 64;
  constexpr int HB = HQ * 8;
  const int64_t tps = ((T + nsplit - 1) / nsplit + DWG_TT - 1) / DWG_TT * DWG_TT;
  dim3 g2((ss.H + HB - 1) / HB, nsplit);
  dwg_partial_kernel<EM><<<g2, HQ * (EM / JT), 0, s>>>(static_cast<const bf16*>(x), dl, T, ss.H, ss.E, tps,
                                            partial);
  const int64_t n = (int64_t)ss.H * ss.E;
  dwg_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(partial, nsplit, n, dwg);
  return cudaGetLastError();
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + WARPS - 1) / WARPS); }

}  // namespace

int gate_bwd_splits(int64_t T) {
  int64_t s = T / 128;
  if (s < 1) s = 1;
  if (s > 128) s = 128;
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
  if (ss.E <= 4) return GB(4, 2, 16);
  if (ss.E <= 8) return GB(8, 2, 16);
  if (ss.E <= 16) return GB(16, 1, 16);
  if (ss.E <= 32) return GB(32, 1, 16);
  return GB(64, 1, 8);
#undef GB
}

}  // namespace moe
