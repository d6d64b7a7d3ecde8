// gate_bwd.cu — B10 on tensor cores (legacy warp MMA; the contractions are tiny):
//   dl_tj = dp_t p_t (delta_{j e*} - softmax(l_t)_j)          (kept tokens; 0 if dropped)
//   dx_t  = dS[row(t)] + sum_j dl_tj Wg[:, j]                   (0 if dropped)
//   dWg   = sum_t x_t^T dl_t                                     (deterministic split-K)
// dl and Wg are fp32; each is split into bf16 hi + lo so the products carry ~16
// mantissa bits (relative error ~2^-17 per term, far inside the 1e-2 gradient
// tolerance); x is exact bf16. (The forward gate's contraction, which decides the
// routing, uses a three-term split of Wg instead: route.cu.)
#include <atomic>
#include <cstdlib>
#include <cuda.h>

#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {


// ------------------------------------------------------------------ Wg -> B' fragments
// B'[k][h] for k in [0, 3*EPK): block 0 = hi(Wg), 1 = hi(Wg), 2 = lo(Wg) (paired with
// A' = [hi(dl) | lo(dl) | hi(dl)]). Packed per (n-tile, k-step) in m16n8k16 B-fragment
// order: word (nt*KS + ks)*64 + lane*2 + {0,1} = {b0, b1} of lane.
__global__ void wg_pack_kernel(const float* __restrict__ wg, int H, int E, int EPK,
                               uint32_t* __restrict__ packed) {
  const int KS = 3 * EPK / 16;
  const int ntiles = H / 8;
  const int64_t n = (int64_t)ntiles * KS * 32;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int lane = (int)(i & 31);
  const int ks = (int)((i >> 5) % KS);
  const int nt = (int)((i >> 5) / KS);
  const int g = lane >> 2, tig = lane & 3;
  const int h = nt * 8 + g;
  auto val = [&](int k) -> bf16 {
    const int blk = k / EPK, j = k % EPK;
    const float v = (j < E) ? wg[(size_t)h * E + j] : 0.f;
    bf16 hi, lo;
    split_bf16(v, hi, lo);
    return blk == 2 ? lo : hi;
  };
  const int k0 = 16 * ks + 2 * tig;
  packed[i * 2] = pack2(val(k0), val(k0 + 1));
  packed[i * 2 + 1] = pack2(val(k0 + 8), val(k0 + 9));
}

// ------------------------------------------------------------------ dl, grow
// Warp per token, every token in flight at once: dl_tj from the saved logits (softmax
// backward; top-2 through the renormalised weights w_k = s_ek / (s_e1 + s_e2), R22; + the
// aux-loss term, R21) with lane j holding experts j, j + 32, and grow [T][KC] = the
// slot-space row of each kept choice (-1 if dropped). The dx kernel below reads both
// instead of recomputing the softmax in every h slice.
template <int EP, int KC>
__global__ void __launch_bounds__(256)
    gate_dl_kernel(const float* __restrict__ logits, const int32_t* __restrict__ expert,
                   const int32_t* __restrict__ slot, const float* __restrict__ prob, const float* __restrict__ dp,
                   SlotSpace ss, int64_t T, float* __restrict__ dl_out, int32_t* __restrict__ grow,
                   const float* __restrict__ aux_f, float aux_scale, bf16* __restrict__ a_tok,
                   int32_t* __restrict__ dwg_cnt, int ncnt) {
  constexpr int JL = EP > 32 ? 2 : 1;  // experts per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = ss.E;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (a_tok && blockIdx.x == 0 && threadIdx.x < ncnt) dwg_cnt[threadIdx.x] = 0;  // dwg_tc's split counters
  if (t >= T) return;
  const float* lg = logits + (size_t)t * E;
  float l[JL], m = -3.402823e38f;
#pragma unroll
  for (int i = 0; i < JL; ++i) {
    const int j = lane + 32 * i;
    l[i] = j < E ? lg[j] : -3.402823e38f;
    m = fmaxf(m, l[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ex[JL], den = 0.f;
#pragma unroll
  for (int i = 0; i < JL; ++i) {
    ex[i] = lane + 32 * i < E ? expf(l[i] - m) : 0.f;
    den += ex[i];
  }
  den = warp_sum(den);
  const float inv = 1.f / den;
  float fs = 0.f;  // sum_e f_e s_te (aux loss)
  if (aux_f) {
#pragma unroll
    for (int i = 0; i < JL; ++i)
      if (lane + 32 * i < E) fs += aux_f[lane + 32 * i] * (ex[i] * inv);
    fs = warp_sum(fs);
  }
  float c1, c2 = 0.f;
  int e1, e2 = -1;
  if (KC == 2) {
    // dL/ds_e1 = s2 (dw1 - dw2) / S^2, dL/ds_e2 = s1 (dw2 - dw1) / S^2 (dw = dp, 0 if dropped)
    e1 = expert[2 * t];
    e2 = expert[2 * t + 1];
    const float s1 = expf(lg[e1] - m) * inv, s2 = expf(lg[e2] - m) * inv;
    const float S = s1 + s2, dw1 = dp[2 * t], dw2 = dp[2 * t + 1];
    c1 = s1 * s2 * (dw1 - dw2) / (S * S);
    c2 = s2 * s1 * (dw2 - dw1) / (S * S);
  } else {
    e1 = expert[t];
    c1 = slot[t] >= 0 ? dp[t] * prob[t] : 0.f;  // dropped: only the aux term
  }
#pragma unroll
  for (int i = 0; i < JL; ++i) {
    const int j = lane + 32 * i;
    if (j < E) {
      const float sj = ex[i] * inv;
      float v = c1 * ((j == e1 ? 1.f : 0.f) - sj);
      if (KC == 2) v += c2 * ((j == e2 ? 1.f : 0.f) - sj);
      if (aux_f) v += aux_scale * sj * (aux_f[j] - fs);
      dl_out[(size_t)t * E + j] = v;
    }
  }
  if (EP <= 32 && a_tok) {
    // dwg_tc's B operand, token order: [hi(dl) | lo(dl) | 0] (EP columns per block, 64 wide)
    const int j = lane;
    float v = 0.f;
    if (j < E) v = dl_out[(size_t)t * E + j];
    bf16 hi, lo;
    split_bf16(v, hi, lo);
    bf16* ar = a_tok + (size_t)t * 64;
    if (j < EP) {
      ar[j] = hi;
      ar[EP + j] = lo;
    }
    if (2 * EP + j < 64) ar[2 * EP + j] = __float2bfloat16_rn(0.f);
  }
  if (lane < KC) {
    const int sl = slot[t * KC + lane];
    int32_t r = -1;
    if (sl >= 0) {
      const int64_t tt = sl / ss.Cs, cs = sl - tt * ss.Cs;
      r = (int32_t)((tt * E + expert[t * KC + lane]) * ss.Cs + cs);
    }
    grow[t * KC + lane] = r;
  }
}

// ------------------------------------------------------------------ dx (+ dl)
// CTA = 4 warps; warp w owns one m-tile of 16 tokens. It builds the A' fragments
// of its tokens (softmax recomputed from the saved logits; lane 4g+tig covers
// tokens g, g+8 and experts 16kk + 2tig + {0,1,8,9}), writes dl [T][E] fp32 for
// dWg, then walks H in 64-wide chunks: 8 n-tiles x KS MMAs, the fp32 results are
// staged in a per-warp shared tile [16][64] and re-read as 16-byte row pieces so
// dS[row(t)] is added and dx stored with coalesced 16-byte accesses.
// KC = 2 (top-2, R22): two dS rows per token and the gate gradient through the
// renormalised weights w_k = s_ek / (s_e1 + s_e2).
constexpr int DX_WARPS = 4;
template <int EPK, int KC>
__global__ void __launch_bounds__(DX_WARPS * 32)
    gate_bwd_dx_mma_kernel(const bf16* __restrict__ dS, const uint32_t* __restrict__ wpk,
                           const float* __restrict__ dl, const int32_t* __restrict__ grow, SlotSpace ss,
                           int64_t T, bf16* __restrict__ dx, bool aux) {
  constexpr int KK = EPK / 16;  // k-steps per block of A'
  constexpr int KS = 3 * KK;
  __shared__ __align__(16) float stage[DX_WARPS][16][64 + 4];
  extern __shared__ __align__(16) uint32_t wsm[];  // this CTA's B' fragments
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int E = ss.E, H = ss.H;
  // H is split over gridDim.y CTAs (more warps in flight for this HBM-bound pass)
  const int ntiles_all = H / 8;
  const int per = ((ntiles_all + gridDim.y - 1) / gridDim.y + 7) & ~7;
  const int nt_begin = blockIdx.y * per;
  const int nt_end = nt_begin + per < ntiles_all ? nt_begin + per : ntiles_all;
  {
    const int nwords = (nt_end - nt_begin) * KS * 64;
    const uint4* src = reinterpret_cast<const uint4*>(wpk + (size_t)nt_begin * KS * 64);
    for (int i = threadIdx.x; i < nwords / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(wsm)[i] = __ldg(src + i);
  }
  __syncthreads();

  const int64_t nblocks = (T + 16 * DX_WARPS - 1) / (16 * DX_WARPS);
  for (int64_t blkid = blockIdx.x; blkid < nblocks; blkid += gridDim.x) {
  const int64_t t0 = (blkid * DX_WARPS + warp) * 16;
  uint32_t afr[KS][4];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int64_t t = t0 + g + 8 * half;
    float dlv[KK][4];  // j = 16 kk + 2 tig + {0, 1, 8, 9}, from gate_dl_kernel
#pragma unroll
    for (int kk = 0; kk < KK; ++kk)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 16 * kk + 2 * tig + (q & 1) + 8 * (q >> 1);
        dlv[kk][q] = (t < T && j < E) ? __ldg(dl + (size_t)t * E + j) : 0.f;
      }
    // A' fragments: a0/a2 rows g (half 0), a1/a3 rows g+8 (half 1)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int blk = ks / KK, kk = ks % KK;
      bf16 h0, l0, h1, l1, h2, l2, h3, l3;
      split_bf16(dlv[kk][0], h0, l0);
      split_bf16(dlv[kk][1], h1, l1);
      split_bf16(dlv[kk][2], h2, l2);
      split_bf16(dlv[kk][3], h3, l3);
      afr[ks][half] = blk == 1 ? pack2(l0, l1) : pack2(h0, h1);      // cols 2tig, 2tig+1
      afr[ks][2 + half] = blk == 1 ? pack2(l2, l3) : pack2(h2, h3);  // cols 2tig+8, 2tig+9
    }
  }
  // per-lane row pieces for the coalesced pass: piece p = lane + 32 k (k < 4) of the
  // 16 x 64 tile -> row p / 8, 8 columns at 8 * (p % 8)
  size_t rowoff[4][KC];
  bool kept[4][KC], valid[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = (lane + 32 * k) >> 3;
    const int64_t t = t0 + r;
    valid[k] = t < T;
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int32_t gr = valid[k] ? __ldg(grow + t * KC + c) : -1;
      kept[k][c] = gr >= 0;
      rowoff[k][c] = kept[k][c] ? (size_t)gr * H : 0;
    }
  }

  const int ntiles = nt_end;
  auto load_ds = [&](int n0, uint4 (&dsv)[4][KC]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 8 * ((lane + 32 * k) & 7);
      const int h = 8 * n0 + c;
#pragma unroll
      for (int q = 0; q < KC; ++q)
        dsv[k][q] = (kept[k][q] && n0 < ntiles && h < 8 * ntiles) ? ld_nc_v4(dS + rowoff[k][q] + h)
                                                                   : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 dsn[4][KC];
  load_ds(nt_begin, dsn);
  for (int n0 = nt_begin; n0 < ntiles; n0 += 8) {
    uint4 dsv[4][KC];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < KC; ++q) dsv[k][q] = dsn[k][q];
    load_ds(n0 + 8, dsn);  // next chunk's dS in flight during this chunk's MMAs
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int nt = n0 + j;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (nt < ntiles) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint2 v = *reinterpret_cast<const uint2*>(wsm + ((nt - nt_begin) * KS + ks) * 64 + lane * 2);
          mma_bf16_16816(acc, afr[ks], v.x, v.y);
        }
      }
      stage[warp][g][8 * j + 2 * tig] = acc[0];
      stage[warp][g][8 * j + 2 * tig + 1] = acc[1];
      stage[warp][g + 8][8 * j + 2 * tig] = acc[2];
      stage[warp][g + 8][8 * j + 2 * tig + 1] = acc[3];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int p = lane + 32 * k, r = p >> 3, c = 8 * (p & 7);
      const int h = 8 * n0 + c;
      if (!valid[k] || h >= 8 * ntiles) continue;
      const float4 g0 = *reinterpret_cast<const float4*>(&stage[warp][r][c]);
      const float4 g1 = *reinterpret_cast<const float4*>(&stage[warp][r][c + 4]);
      uint4 o = make_uint4(0, 0, 0, 0);
      if (KC == 2) {  // dS rows of the kept choices (zeros otherwise) + the gate term
        float sv[8];
        const uint32_t a0[4] = {dsv[k][0].x, dsv[k][0].y, dsv[k][0].z, dsv[k][0].w};
        const uint32_t a1[4] = {dsv[k][KC - 1].x, dsv[k][KC - 1].y, dsv[k][KC - 1].z, dsv[k][KC - 1].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 u0 = unpack_bf16x2(a0[q]), u1 = unpack_bf16x2(a1[q]);
          sv[2 * q] = u0.x + u1.x;
          sv[2 * q + 1] = u0.y + u1.y;
        }
        o = make_uint4(pack_bf16x2(sv[0] + g0.x, sv[1] + g0.y), pack_bf16x2(sv[2] + g0.z, sv[3] + g0.w),
                       pack_bf16x2(sv[4] + g1.x, sv[5] + g1.y), pack_bf16x2(sv[6] + g1.z, sv[7] + g1.w));
      } else if (kept[k][0]) {
        const float2 s0 = unpack_bf16x2(dsv[k][0].x), s1 = unpack_bf16x2(dsv[k][0].y);
        const float2 s2 = unpack_bf16x2(dsv[k][0].z), s3 = unpack_bf16x2(dsv[k][0].w);
        o = make_uint4(pack_bf16x2(s0.x + g0.x, s0.y + g0.y), pack_bf16x2(s1.x + g0.z, s1.y + g0.w),
                       pack_bf16x2(s2.x + g1.x, s2.y + g1.y), pack_bf16x2(s3.x + g1.z, s3.y + g1.w));
      } else if (aux) {  // dropped token: only the aux-loss gate gradient
        o = make_uint4(pack_bf16x2(g0.x, g0.y), pack_bf16x2(g0.z, g0.w), pack_bf16x2(g1.x, g1.y),
                       pack_bf16x2(g1.z, g1.w));
      }
      st_v4(dx + (size_t)(t0 + r) * H + h, o);
    }
    __syncwarp();
  }
  }
}

// ------------------------------------------------------------------ dWg partials
// D[e'][h] = sum_t A[e'][t] B[t][h], A = [hi(dl) | lo(dl)]^T (2*EP rows), B = x.
// CTA = 8 warps over HB = 8*NT*8 columns of h, one token split; tiles of 32 tokens
// staged in shared memory (register-prefetched one tile ahead), fragments via
// ldmatrix.trans. dWg[h][e] = D[e][h] + D[EP+e][h] is written as a partial.
constexpr int DW_TT = 32;
template <int EP>
__global__ void __launch_bounds__(256)
    dwg_mma_kernel(const bf16* __restrict__ x, const float* __restrict__ dl, int64_t T, int H, int E,
                   int64_t tok_per_split, float* __restrict__ partial) {
  constexpr int M2 = 2 * EP;            // rows of A (hi | lo)
  constexpr int MT = (M2 + 15) / 16;    // m-tiles
  constexpr int MROWS = MT * 16;
  constexpr int NT = EP <= 32 ? 4 : 2;  // n-tiles per warp
  constexpr int HB = 8 * NT * 8;        // h per CTA
  constexpr int SA = MROWS + 8;         // dl_s row stride (bf16 elements), +16 B pad
  constexpr int SB = HB + 8;            // x_s row stride
  __shared__ __align__(16) bf16 dl_s[DW_TT][SA];
  __shared__ __align__(16) bf16 x_s[DW_TT][SB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hb = blockIdx.x * HB;
  const int64_t t_begin = (int64_t)blockIdx.y * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > T) t_end = T;

  constexpr int XV = DW_TT * HB / 8 / 256;  // 16-byte x vectors per thread per tile
  constexpr int DV = (DW_TT * EP + 255) / 256;
  uint4 xr[XV];
  float dr[DV];
  auto load_tile = [&](int64_t tb) {
#pragma unroll
    for (int k = 0; k < XV; ++k) {
      const int i = threadIdx.x + k * 256;
      const int tt = i / (HB / 8), v = i % (HB / 8);
      const int64_t t = tb + tt;
      const int h = hb + 8 * v;
      xr[k] = (t < t_end && h < H) ? ld_nc_v4(x + (size_t)t * H + h) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < DV; ++k) {
      const int i = threadIdx.x + k * 256;
      const int tt = i / EP, j = i % EP;
      const int64_t t = tb + tt;
      dr[k] = (i < DW_TT * EP && t < t_end && j < E) ? __ldg(dl + (size_t)t * E + j) : 0.f;
    }
  };
  float acc[MT][NT][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
  // rows MROWS > 2*EP (only when EP == 4) stay zero
  for (int i = threadIdx.x; i < DW_TT * SA; i += 256) (&dl_s[0][0])[i] = __float2bfloat16_rn(0.f);
  if (t_begin < t_end) load_tile(t_begin);
  for (int64_t tb = t_begin; tb < t_end; tb += DW_TT) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < XV; ++k) {
      const int i = threadIdx.x + k * 256;
      const int tt = i / (HB / 8), v = i % (HB / 8);
      *reinterpret_cast<uint4*>(&x_s[tt][8 * v]) = xr[k];
    }
#pragma unroll
    for (int k = 0; k < DV; ++k) {
      const int i = threadIdx.x + k * 256;
      if (i < DW_TT * EP) {
        const int tt = i / EP, j = i % EP;
        bf16 hi, lo;
        split_bf16(dr[k], hi, lo);
        dl_s[tt][j] = hi;
        dl_s[tt][EP + j] = lo;
      }
    }
    __syncthreads();
    if (tb + DW_TT < t_end) load_tile(tb + DW_TT);
#pragma unroll
    for (int ks = 0; ks < DW_TT / 16; ++ks) {
      const int mi = lane >> 3, r = lane & 7;
      uint32_t afr[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int t = 16 * ks + r + 8 * (mi >> 1);
        const int e = 16 * mt + 8 * (mi & 1);
        ldmatrix_x4_trans(afr[mt], smem_u32(&dl_s[t][e]));
      }
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int t = 16 * ks + r + 8 * (mi & 1);
        const int hcol = warp * NT * 8 + 16 * np + 8 * (mi >> 1);
        uint32_t bfr[4];
        ldmatrix_x4_trans(bfr, smem_u32(&x_s[t][hcol]));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma_bf16_16816(acc[mt][2 * np], afr[mt], bfr[0], bfr[1]);
          mma_bf16_16816(acc[mt][2 * np + 1], afr[mt], bfr[2], bfr[3]);
        }
      }
    }
  }
  // epilogue: rows e' = 16 mt + g (+8); cols h = hb + warp*NT*8 + 8 nt + 2 tig (+1)
  const int g = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int er = 16 * mt + g + 8 * half;  // row of D
      if (er >= EP) continue;                 // lo rows are folded into their hi row
      const int elo = er + EP;
      const int mlo = elo / 16, hlo = (elo % 16) >= 8 ? 1 : 0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int h = hb + warp * NT * 8 + 8 * nt + 2 * tig;
        if (er >= E || h >= H) continue;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v = acc[mt][nt][2 * half + c];
#pragma unroll
          for (int m2 = 0; m2 < MT; ++m2)
            if (m2 == mlo) v += hlo ? acc[m2][nt][2 + c] : acc[m2][nt][c];
          partial[((size_t)blockIdx.y * H + h + c) * E + er] = v;
        }
      }
    }
}

__global__ void dwg_reduce2_kernel(const float* __restrict__ partial, int nsplit, int64_t n,
                                   float* __restrict__ dwg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int k = 0; k < nsplit; ++k) s += partial[(size_t)k * n + i];
  dwg[i] = s;
}

// ------------------------------------------------------------------ fused one-GPU B1 + B10 head
// One launch replaces combine_bwd + zero_empty + gate_dl + gate_ext_a/b + zero_dropped
// (top-1, one GPU, E <= 16; slot space == expert space, row r = e * C + c). Warp work items:
//   [0, E*C)           slot row r: kept -> t = tok_of[r]: dp = <dy_t, O_r> (fp32),
//                      dO_r = bf16(p_t dy_t), then lanes j < E: dl_tj = dp p_t (d_{j e*} - s_tj)
//                      (fp32, for dWg) and the K-extension row a_ext[r] = [hi | lo | hi | 0](dl_t);
//                      empty -> dO_r = 0, a_ext[r] = 0
//   next T/32          32 tokens per warp: dropped tokens get dl_t = 0 and dx_t = 0 (B5's
//                      scatter writes only kept rows)
//   next 16*H/256      b_ext = [hi(Wg)^T ; hi(Wg)^T ; lo(Wg)^T ; 0], 256 h of one j per warp
constexpr int CBG_WARPS = 8;
__global__ void __launch_bounds__(CBG_WARPS * 32)
    combine_bwd_gate_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ O,
                            const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                            const float* __restrict__ prob, const float* __restrict__ logits,
                            const int32_t* __restrict__ tok_of, const int32_t* __restrict__ count,
                            const float* __restrict__ wg, int64_t T, int H, int E, int64_t C,
                            bf16* __restrict__ dO, float* __restrict__ dl, bf16* __restrict__ a_ext,
                            bf16* __restrict__ b_ext, bf16* __restrict__ dx, int32_t* __restrict__ dwg_cnt,
                            int ncnt) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0)  // split-K counters of the dWg launch that follows (stream order)
    for (int i = threadIdx.x; i < ncnt; i += blockDim.x) dwg_cnt[i] = 0;
  int64_t w = (int64_t)blockIdx.x * CBG_WARPS + (threadIdx.x >> 5);
  const int64_t rows = (int64_t)E * C;
  const int nv = H / 8;
  if (w < rows) {
    const int e = (int)(w / C);
    const int64_t c = w - (int64_t)e * C;
    bf16* dst = dO + (size_t)w * H;
    bf16* arow = a_ext + (size_t)w * 64;
    if (c >= count[e]) {
      for (int v = lane; v < nv; v += 32) st_v4(dst + (size_t)v * 8, make_uint4(0, 0, 0, 0));
      if (lane < 8) st_v4(arow + lane * 8, make_uint4(0, 0, 0, 0));
      return;
    }
    const int t = tok_of[w];
    const float p = prob[t];
    const bf16* dyr = dy + (size_t)t * H;
    const bf16* orow = O + (size_t)w * H;
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
        const uint32_t wa[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
        const uint32_t wb[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 fa = unpack_bf16x2(wa[k]), fb = unpack_bf16x2(wb[k]);
          acc = fmaf(fa.x, fb.x, acc);
          acc = fmaf(fa.y, fb.y, acc);
          o[k] = pack_bf16x2(p * fa.x, p * fa.y);
        }
        if (v < nv) st_v4(dst + (size_t)v * 8, make_uint4(o[0], o[1], o[2], o[3]));
      }
    }
    const float dp = warp_sum(acc);
    // softmax of the saved logits over lanes j < E (E <= 16 on this path)
    const float lj = lane < E ? logits[(size_t)t * E + lane] : -3.402823e38f;
    float m = lj;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float ex = lane < E ? expf(lj - m) : 0.f;
    const float den = warp_sum(ex);
    const float d = lane < E ? dp * p * ((lane == expert[t] ? 1.f : 0.f) - ex / den) : 0.f;
    if (lane < E) dl[(size_t)t * E + lane] = d;
    if (lane < 16) {
      bf16 hi, lo;
      split_bf16(d, hi, lo);
      arow[lane] = hi;
      arow[16 + lane] = lo;
      arow[32 + lane] = hi;
      arow[48 + lane] = __float2bfloat16_rn(0.f);
    }
    return;
  }
  w -= rows;
  const int64_t tw = (T + 31) / 32;
  if (w < tw) {
    const int64_t t = w * 32 + lane;
    const bool dropped = t < T && slot[t] < 0;
    uint32_t mask = __ballot_sync(0xffffffffu, dropped);
    if (dropped)
      for (int j = 0; j < E; ++j) dl[(size_t)t * E + j] = 0.f;
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      bf16* xr = dx + (size_t)(w * 32 + l) * H;
      for (int v = lane; v < nv; v += 32) st_v4(xr + (size_t)v * 8, make_uint4(0, 0, 0, 0));
    }
    return;
  }
  w -= tw;
  const int64_t hb = (H + 255) / 256;
  if (w >= 16 * hb) return;
  const int j = (int)(w / hb);
  const int h0 = (int)(w - (int64_t)j * hb) * 256 + lane * 8;
  if (h0 >= H) return;
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bf16 h2[2], l2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) split_bf16(j < E ? wg[(size_t)(h0 + 2 * i + u) * E + j] : 0.f, h2[u], l2[u]);
    hw[i] = pack2(h2[0], h2[1]);
    lw[i] = pack2(l2[0], l2[1]);
  }
  const uint4 vh = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  st_v4(b_ext + (size_t)j * H + h0, vh);
  st_v4(b_ext + (size_t)(16 + j) * H + h0, vh);
  st_v4(b_ext + (size_t)(32 + j) * H + h0, make_uint4(lw[0], lw[1], lw[2], lw[3]));
  st_v4(b_ext + (size_t)(48 + j) * H + h0, make_uint4(0, 0, 0, 0));
}

// ------------------------------------------------------------------ dWg on the tensor cores
// One GPU, top-1, E <= 16: dWg = sum_t x_t^T dl_t = sum over kept slot rows r of
// X_r^T dl_tok(r) (dl is zero for dropped tokens), with X the dispatched rows [E*C][H]
// (expert space) and the K-extension rows a_ext [E*C][64] = [hi(dl) | lo(dl) | hi | 0]
// that combine_bwd_gate already wrote. D[h][n] = sum_r X[r][h] a_ext[r][n] is a
// tcgen05 GEMM with M = 128 h (A = X, MN-major), N = 64 (B = a_ext, MN-major), K = rows,
// and dWg[h][j] = D[h][j] + D[h][16 + j]. Split-K over nsplit CTAs per 128-row h tile
// (CTA = split * mtiles + tile, so CTAs running together read the same rows); each
// writes its partial, and the last CTA of a tile (counter zeroed by combine_bwd_gate)
// sums the partials in split order: deterministic, one launch.
namespace dwtc {
constexpr int A_BYTES = 128 * 64 * 2;
constexpr int B_BYTES = 64 * 64 * 2;
constexpr int STAGES = 8;
constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 + 256;
constexpr int THREADS = 192;

__device__ __forceinline__ void tmem_ld16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
}

__device__ __forceinline__ uint64_t mn_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(8192 >> 4) << 16;  // LBO: next 64-wide MN block
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8 K-rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

template <int EP>
__global__ void __launch_bounds__(THREADS, 1)
    dwg_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t rows,
                  int H, int E, int mtiles, int nsplit, float* __restrict__ partial, int32_t* __restrict__ cnt,
                  float* __restrict__ dwg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * (A_BYTES + B_BYTES));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (int)(blockIdx.x % mtiles), split = (int)(blockIdx.x / mtiles);
  const int h0 = mt * 128;
  const int KB = (int)((rows + 63) / 64);
  const int per = (KB + nsplit - 1) / nsplit;
  const int kb0 = split * per;
  const int kb1 = kb0 + per < KB ? kb0 + per : KB;
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[STAGES + s]), 1);
    }
    mbar_init(smem_u32(&bars[2 * STAGES]), 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent

  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int stage = i % STAGES;
        const uint32_t phase = (uint32_t)(i / STAGES) & 1;
        mbar_wait(smem_u32(&bars[STAGES + stage]), phase ^ 1);
        const uint32_t full = smem_u32(&bars[stage]);
        mbar_arrive_expect_tx(full, A_BYTES + B_BYTES);
        const uint32_t a = smem_u32(smem + stage * (A_BYTES + B_BYTES));
        const int r0 = (kb0 + i) * 64;
        tma_load_3d(a, &tmA, full, h0, r0, 0);
        tma_load_3d(a + 8192, &tmA, full, h0 + 64, r0, 0);
        tma_load_3d(a + A_BYTES, &tmB, full, 0, r0, 0);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                                 ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int i = 0; i < nkb; ++i) {
        const int stage = i % STAGES;
        mbar_wait(smem_u32(&bars[stage]), (uint32_t)(i / STAGES) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + stage * (A_BYTES + B_BYTES));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          tc_mma_f16(tmem, mn_desc(a + j * 2048), mn_desc(a + A_BYTES + j * 2048), idesc, (i | j) ? 1u : 0u);
        tc_commit(smem_u32(&bars[STAGES + stage]));
      }
      if (nkb > 0) tc_commit(smem_u32(&bars[2 * STAGES]));
    }
    __syncwarp();
  } else {
    // epilogue warps 0-3: TMEM lane = h row of the tile; dWg[h][j] = D[h][j] + D[h][EP + j]
    // (a_ext columns [hi(dl) | lo(dl)], EP = 16 or 32)
    const int hl = warp * 32 + lane;
    const int h = h0 + hl;
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    if (nkb > 0) {
      mbar_wait(smem_u32(&bars[2 * STAGES]), 0);
      tc_fence_after();
    }
    float* prow = partial + ((size_t)split * H + (h < H ? h : 0)) * E;
#pragma unroll
    for (int c = 0; c < EP; c += 16) {
      float v[16];
      if (nkb > 0) {
        uint32_t hi[16], lo[16];
        tmem_ld16(ta + c, hi);
        tmem_ld16(ta + EP + c, lo);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(hi[j]) + __uint_as_float(lo[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
      if (h < H)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c + j < E) prow[c + j] = v[j];
    }
    __threadfence();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 0) last = atomicAdd(&cnt[mt], 1) == nsplit - 1;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (last) {  // every split of this h tile is in: sum in split order
      __threadfence();
      if (h < H) {
        // sum over splits in split order per j; the loads of several splits are issued
        // together (a load -> add chain per (j, split) made this tail ~half the kernel)
        float acc[EP];
#pragma unroll
        for (int j = 0; j < EP; ++j) acc[j] = 0.f;
#pragma unroll 4
        for (int sp = 0; sp < nsplit; ++sp) {
          const float* pr = partial + ((size_t)sp * H + h) * E;
#pragma unroll
          for (int j = 0; j < EP; ++j)
            if (j < E) acc[j] += __ldcg(pr + j);
        }
#pragma unroll
        for (int j = 0; j < EP; ++j)
          if (j < E) dwg[(size_t)h * E + j] = acc[j];
      }
      if (threadIdx.x == 0) cnt[mt] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64) : "memory");
  }
}
}  // namespace dwtc

template <int EP>
cudaError_t dwg_only(const void* x, const float* dl, int64_t T, int H, int E, float* dwg, float* partial,
                     int nsplit, cudaStream_t s) {
  constexpr int NT = EP <= 32 ? 4 : 2;
  constexpr int HB = 8 * NT * 8;
  const int64_t tps = ((T + nsplit - 1) / nsplit + DW_TT - 1) / DW_TT * DW_TT;
  dim3 g2((H + HB - 1) / HB, nsplit);
  dwg_mma_kernel<EP><<<g2, 256, 0, s>>>(static_cast<const bf16*>(x), dl, T, H, E, tps, partial);
  const int64_t n = (int64_t)H * E;
  dwg_reduce2_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(partial, nsplit, n, dwg);
  return cudaGetLastError();
}

template <int EPK, int EP, int KC>
cudaError_t run(const void* x, const void* dS, const float* wg, const float* logits,
                const int32_t* expert, const int32_t* slot, const float* prob, const float* dp,
                const SlotSpace& ss, int64_t T, void* dx, float* dwg, float* dl, int32_t* grow, float* partial,
                int nsplit, uint32_t* wpk, void* a_tok_scratch, int32_t* dwg_cnt, const float* aux_f, float aux_scale,
                cudaStream_t s) {
  const int H = ss.H, E = ss.E;
  const int KS = 3 * EPK / 16;
  const int64_t npack = (int64_t)(H / 8) * KS * 32;
  wg_pack_kernel<<<(unsigned)((npack + 255) / 256), 256, 0, s>>>(wg, H, E, EPK, wpk);
  const int64_t tb = 16 * DX_WARPS;
  // split H so that the CTA's B' slice (per * KS * 256 bytes) stays small: more CTAs
  // (warps) per SM for this latency-bound gather + tiny-K MMA pass
  const int ntiles = H / 8;
  // measured (emulated EP2 / TP2xEP2, ncu): 48 KiB for E <= 16 (53 vs 57 us at 1.3B),
  // 96 KiB above (76 vs 79 us at 2.7B)
  static const int budget = [] {
    const char* e = getenv("MOE_DX_BUDGET_KB");  // development knob
    return (e ? atoi(e) : (EPK == 16 ? 48 : 96)) * 1024;
  }();
  int hsplit = 1;
  auto slice_bytes = [&](int hs) { return (size_t)(((ntiles + hs - 1) / hs + 7) & ~7) * KS * 256; };
  while (slice_bytes(hsplit) > (size_t)budget && hsplit < ntiles / 8) hsplit *= 2;
  const size_t smem = slice_bytes(hsplit);
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_bwd_dx_mma_kernel<EPK, KC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gate_bwd_dx_mma_kernel<EPK, KC>, DX_WARPS * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t gx = (T + tb - 1) / tb;
  const int64_t cap = ((int64_t)per_sm * sms + hsplit - 1) / hsplit;  // one resident wave, persistent
  if (gx > cap) gx = cap;
  bf16* a_tok = EPK <= 32 ? static_cast<bf16*>(a_tok_scratch) : nullptr;
  gate_dl_kernel<EPK, KC><<<(unsigned)((T + 7) / 8), 256, 0, s>>>(logits, expert, slot, prob, dp, ss, T, dl, grow,
                                                                  aux_f, aux_scale, a_tok, dwg_cnt, (H + 127) / 128);
  gate_bwd_dx_mma_kernel<EPK, KC><<<dim3((unsigned)gx, hsplit), DX_WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(dS), wpk, dl, grow, ss, T, static_cast<bf16*>(dx), aux_f != nullptr);
  if (EPK <= 32)  // dWg on the tensor cores from the token-order [hi | lo](dl) rows (one launch)
    return gate_dwg_tc(x, a_tok, T, H, E, dwg, partial, DWG_TC_SPLITS, dwg_cnt, s);
  constexpr int NT = EP <= 32 ? 4 : 2;
  constexpr int HB = 8 * NT * 8;
  const int64_t tps = ((T + nsplit - 1) / nsplit + DW_TT - 1) / DW_TT * DW_TT;
  dim3 g2((H + HB - 1) / HB, nsplit);
  dwg_mma_kernel<EP><<<g2, 256, 0, s>>>(static_cast<const bf16*>(x), dl, T, H, E, tps, partial);
  const int64_t n = (int64_t)H * E;
  dwg_reduce2_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(partial, nsplit, n, dwg);
  return cudaGetLastError();
}

}  // namespace

size_t gate_bwd_pack_bytes(int H, int E) {
  const int EPK = E <= 16 ? 16 : (E <= 32 ? 32 : 64);
  return (size_t)(H / 8) * (3 * EPK / 16) * 64 * 4;
}

cudaError_t gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                     const int32_t* expert, const int32_t* slot, const float* prob,
                     const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                     float* dl_scratch, int32_t* grow, float* dwg_partial, int nsplit, void* pack_scratch,
                     void* a_tok_scratch, int32_t* dwg_cnt,
                     const float* aux_f, float aux_coef, cudaStream_t s) {
  if (T <= 0) return cudaMemsetAsync(dwg, 0, sizeof(float) * ss.H * ss.E, s);
  uint32_t* wpk = static_cast<uint32_t*>(pack_scratch);
  // d l_aux / d l_tj = coef * E / T * s_tj (f_j - sum_e f_e s_te)
  const float aux_scale = aux_f ? (float)((double)aux_coef * ss.E / (double)T) : 0.f;
#define RUN(EPK, EP)                                                                                         \
  (ss.K == 2 ? run<EPK, EP, 2>(x, dS, wg, logits, expert, slot, prob, dp, ss, T, dx, dwg, dl_scratch, grow,  \
                               dwg_partial, nsplit, wpk, a_tok_scratch, dwg_cnt, aux_f, aux_scale, s)                                 \
             : run<EPK, EP, 1>(x, dS, wg, logits, expert, slot, prob, dp, ss, T, dx, dwg, dl_scratch, grow,  \
                               dwg_partial, nsplit, wpk, a_tok_scratch, dwg_cnt, aux_f, aux_scale, s))
  if (ss.E <= 8) return RUN(16, 8);  // EP >= 8: a lo row sits in the same thread as its hi row
  if (ss.E <= 16) return RUN(16, 16);
  if (ss.E <= 32) return RUN(32, 32);
  return RUN(64, 64);
#undef RUN
}

cudaError_t combine_bwd_gate(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                             const float* prob, const float* logits, const int32_t* tok_of,
                             const int32_t* count, const float* wg, int64_t T, int H, int E, int64_t C,
                             void* dO, float* dl, void* a_ext, void* b_ext, void* dx, int32_t* dwg_cnt,
                             cudaStream_t s) {
  if (E > 16) return cudaErrorInvalidValue;
  const int64_t items = (int64_t)E * C + (T + 31) / 32 + 16 * ((H + 255) / 256);
  combine_bwd_gate_kernel<<<(unsigned)((items + CBG_WARPS - 1) / CBG_WARPS), CBG_WARPS * 32, 0, s>>>(
      static_cast<const bf16*>(dy), static_cast<const bf16*>(O), expert, slot, prob, logits, tok_of, count, wg,
      T, H, E, C, static_cast<bf16*>(dO), dl, static_cast<bf16*>(a_ext), static_cast<bf16*>(b_ext),
      static_cast<bf16*>(dx), dwg_cnt, (H + 127) / 128);
  return cudaGetLastError();
}

template <int EP>
static cudaError_t dwg_tc_launch(const void* X, const void* a_ext, int64_t rows, int H, int E, float* dwg,
                                 float* partial, int max_split, int32_t* counters, cudaStream_t s) {
  CUtensorMap ta, tb;
  int sms = 0;
  cudaError_t e = tensor_map_bf16(&ta, X, (uint64_t)H, (uint64_t)rows, 64, 64, &sms);
  if (e == cudaSuccess) e = tensor_map_bf16(&tb, a_ext, 64, (uint64_t)rows, 64, 64, &sms);
  if (e != cudaSuccess) return e;
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  if (!attr) {
    e = cudaFuncSetAttribute(dwtc::dwg_tc_kernel<EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, dwtc::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int mtiles = (H + 127) / 128;
  const int kb = (int)((rows + 63) / 64);
  int nsplit = sms / mtiles;                  // one wave
  if (nsplit > (kb + 3) / 4) nsplit = (kb + 3) / 4;  // >= 4 k-blocks per CTA
  if (nsplit > max_split) nsplit = max_split;
  if (nsplit < 1) nsplit = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(mtiles * nsplit));
  cfg.blockDim = dim3(dwtc::THREADS);
  cfg.dynamicSmemBytes = dwtc::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];  // the prologue overlaps the tail of the previous kernel
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dwtc::dwg_tc_kernel<EP>, ta, tb, rows, H, E, mtiles, nsplit, partial, counters,
                            dwg);
}

cudaError_t gate_dwg_tc(const void* X, const void* a_ext, int64_t rows, int H, int E, float* dwg, float* partial,
                        int max_split, int32_t* counters, cudaStream_t s) {
  if (E > 32) return cudaErrorInvalidValue;
  if (rows <= 0) return cudaMemsetAsync(dwg, 0, sizeof(float) * H * E, s);
  return E <= 16 ? dwg_tc_launch<16>(X, a_ext, rows, H, E, dwg, partial, max_split, counters, s)
                 : dwg_tc_launch<32>(X, a_ext, rows, H, E, dwg, partial, max_split, counters, s);
}

cudaError_t gate_dwg(const void* x, const float* dl, int64_t T, int H, int E, float* dwg, float* partial,
                     int nsplit, cudaStream_t s) {
  if (T <= 0) return cudaMemsetAsync(dwg, 0, sizeof(float) * H * E, s);
  if (E <= 8) return dwg_only<8>(x, dl, T, H, E, dwg, partial, nsplit, s);
  if (E <= 16) return dwg_only<16>(x, dl, T, H, E, dwg, partial, nsplit, s);
  if (E <= 32) return dwg_only<32>(x, dl, T, H, E, dwg, partial, nsplit, s);
  return dwg_only<64>(x, dl, T, H, E, dwg, partial, nsplit, s);
}

int gate_bwd_splits(int64_t T) {
  int64_t s = T / 512;
  if (s < 1) s = 1;
  if (s > 32) s = 32;
  return (int)s;
}

}  // namespace moe
