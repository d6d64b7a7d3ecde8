// permute.cu — the HBM-bound steps of the hot path:
//   F3  dispatch      slot-parallel gather x -> capacity-padded slot space
//   F11 combine       token-parallel y_t = sum_k p_tk * O[row(t,k)]  (K = 1, or 2 for top-2)
//   B1  combine_bwd   dp_tk = <dy_t, O[row(t,k)]>, dO[row(t,k)] = p_tk dy_t
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

// Warps [0, rows): one slot row each. With y_zero (one GPU, F11 fused into F7's
// epilogue, which writes only kept tokens' rows) warps [rows, rows + T/32) zero the y
// rows of the dropped tokens among 32 tokens each.
__global__ void __launch_bounds__(WARPS * 32)
    dispatch_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ tok_of,
                    const int32_t* __restrict__ count, SlotSpace ss, int t_lo, int64_t rows,
                    bf16* __restrict__ D, const int32_t* __restrict__ slot, int64_t T,
                    bf16* __restrict__ y_zero) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) {
    const int64_t t = (r - rows) * 32 + lane;
    if (!y_zero || (r - rows) * 32 >= T) return;
    uint32_t mask = __ballot_sync(0xffffffffu, t < T && slot[t] < 0);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      copy_row<true>(nullptr, y_zero + (size_t)((r - rows) * 32 + l) * ss.H, ss.H / 8, lane);
    }
    return;
  }
  const int64_t per_slice = (int64_t)ss.E * ss.Cs;
  const int tt = t_lo + (int)(r / per_slice);
  const int64_t rem = r % per_slice;
  const int e = (int)(rem / ss.Cs);
  const int64_t cs = rem % ss.Cs;
  const int64_t c = (int64_t)tt * ss.Cs + cs;
  bf16* dst = D + ((size_t)(tt * ss.E + e) * ss.Cs + cs) * ss.H;
  const int nv = ss.H / 8;
  if (c < count[e]) {
    const int t = tok_of[(size_t)e * ss.C + c] / ss.K;  // item -> token
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
  const int K = ss.K;
  const int nv = ss.H / 8;
  bf16* dst = y + (size_t)t * ss.H;
  const bf16* src[2] = {nullptr, nullptr};
  float p[2] = {0.f, 0.f};
  int nk = 0;
  for (int k = 0; k < K; ++k) {
    const int s = slot[t * K + k];
    if (s < 0) continue;
    src[nk] = O + slot_row(ss, expert[t * K + k], s);
    p[nk] = prob[t * K + k];
    ++nk;
  }
  if (nk == 0) {
    copy_row<true>(nullptr, dst, nv, lane);
    return;
  }
  constexpr int U = 8;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    uint4 buf[U], buf2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      buf[u] = v < nv ? ld_nc_v4(src[0] + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
      buf2[u] = (nk > 1 && v < nv) ? ld_nc_v4(src[1] + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) {
        uint32_t w[4] = {buf[u].x, buf[u].y, buf[u].z, buf[u].w};
        const uint32_t w2[4] = {buf2[u].x, buf2[u].y, buf2[u].z, buf2[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = unpack_bf16x2(w[k]);
          float2 r = make_float2(p[0] * f.x, p[0] * f.y);
          if (nk > 1) {  // second choice (top-2): fp32 sum, one rounding
            const float2 f2 = unpack_bf16x2(w2[k]);
            r = make_float2(fmaf(p[1], f2.x, r.x), fmaf(p[1], f2.y, r.y));
          }
          w[k] = pack_bf16x2(r.x, r.y);
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
  for (int kc = 0; kc < ss.K; ++kc) {
  const int64_t it = t * ss.K + kc;
  const int s = slot[it];
  if (s < 0) {
    if (lane == 0) dp[it] = 0.f;
    continue;
  }
  const size_t row = slot_row(ss, expert[it], s);
  const int tt = (int)(s / ss.Cs);
  const bool mine = tt >= t_lo && tt < t_hi;
  const float p = prob[it];
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
  if (lane == 0) dp[it] = acc;
  }
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


// ---------------------------------------------------------------- fused peer variants
__device__ __forceinline__ uint8_t* peer_row(const PeerDst& pd, int tt, int e, int64_t cs,
                                             const SlotSpace& ss, int t2) {
  const int ep2 = e / pd.El, el = e % pd.El;
  const int r = (pd.d * pd.Gep + ep2) * pd.Gt + t2;
  uint8_t* base = static_cast<uint8_t*>(pd.table[(size_t)r * pd.nwin + pd.win]);
  return base + ((((size_t)el * pd.Gt + tt) * pd.Gep + pd.ep) * ss.Cs + cs) * ss.H * 2;
}

// Row offset of slot (tt, e, cs) in the expert-space window (the same on every TP rank).
__device__ __forceinline__ size_t peer_off(const PeerDst& pd, int tt, int e, int64_t cs, const SlotSpace& ss) {
  const int el = e % pd.El;
  return ((((size_t)el * pd.Gt + tt) * pd.Gep + pd.ep) * ss.Cs + cs) * ss.H * 2;
}

// Destinations of one row: G_t TP ranks (DTD fold), one multicast store when the owner
// group is this rank's own and a multicast mapping exists (MOE_F_NVLS direct), or the
// same-t rank (vanilla / two-step NVLS). Returns the count; *mc says "multicast".
__device__ __forceinline__ int row_dsts(const PeerDst& pd, int tt, int e, int64_t cs, const SlotSpace& ss,
                                        bf16* (&dsts)[8], bool* mc) {
  *mc = pd.dtd && pd.mc && e / pd.El == pd.ep;
  if (*mc) {
    dsts[0] = reinterpret_cast<bf16*>(static_cast<uint8_t*>(pd.mc) + peer_off(pd, tt, e, cs, ss));
    return 1;
  }
  const int nd = pd.dtd ? pd.Gt : 1;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    dsts[k] = k < nd ? reinterpret_cast<bf16*>(peer_row(pd, tt, e, cs, ss, pd.dtd ? k : pd.t)) : nullptr;
  return nd;
}

// One warp per slot row: the x row (or zeros) is read once and stored to every
// destination rank (1 for vanilla, G_t for DTD, one multicast store for the own group
// under MOE_F_NVLS) with 16-byte stores over NVLink.
__global__ void __launch_bounds__(WARPS * 32)
    dispatch_peer_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ tok_of,
                         const int32_t* __restrict__ count, SlotSpace ss, int t_lo, int64_t rows,
                         PeerDst pd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t per_slice = (int64_t)ss.E * ss.Cs;
  const int tt = t_lo + (int)(r / per_slice);
  const int64_t rem = r % per_slice;
  const int e = (int)(rem / ss.Cs);
  const int64_t cs = rem % ss.Cs;
  const int64_t c = (int64_t)tt * ss.Cs + cs;
  const int nv = ss.H / 8;
  const bool full = c < count[e];
  const bf16* src = full ? x + (size_t)(tok_of[(size_t)e * ss.C + c] / ss.K) * ss.H : nullptr;
  constexpr int MAXD = 8;  // destination rows resolved once per row (G_t <= 8)
  bf16* dsts[MAXD];
  bool mc;
  const int nd = row_dsts(pd, tt, e, cs, ss, dsts, &mc);
  constexpr int U = 8;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    uint4 buf[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 32 + lane;
      buf[u] = (full && v < nv) ? ld_nc_v4(src + (size_t)v * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      if (k >= nd) break;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nv) {
          if (mc) st_mc_v4(dsts[k] + (size_t)v * 8, buf[u]);
          else st_v4(dsts[k] + (size_t)v * 8, buf[u]);
        }
      }
    }
  }
  __threadfence_system();
}

// Token-parallel: dp_t = <dy_t, O[row(t)]>; for kept tokens whose slot is in
// slices [t_lo, t_hi), the row p_t dy_t is stored to every destination rank.
__global__ void __launch_bounds__(WARPS * 32)
    combine_bwd_peer_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ O,
                            const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                            const float* __restrict__ prob, SlotSpace ss, int64_t T, int t_lo,
                            int t_hi, float* __restrict__ dp, PeerDst pd) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= T) return;
  for (int kc = 0; kc < ss.K; ++kc) {
  const int64_t it = t * ss.K + kc;
  const int s = slot[it];
  if (s < 0) {
    if (lane == 0) dp[it] = 0.f;
    continue;
  }
  const int e = expert[it];
  const size_t row = slot_row(ss, e, s);
  const int tt = (int)(s / ss.Cs);
  const int64_t cs = s - (int64_t)tt * ss.Cs;
  const bool mine = tt >= t_lo && tt < t_hi;
  const float p = prob[it];
  const bf16* dyr = dy + (size_t)t * ss.H;
  const bf16* orow = O + row;
  const int nv = ss.H / 8;
  constexpr int MAXD = 8;
  bf16* dsts[MAXD];
  bool mc = false;
  const int nd = mine ? row_dsts(pd, tt, e, cs, ss, dsts, &mc) : 0;
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
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t wa[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
      uint32_t wb[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 fa = unpack_bf16x2(wa[k]), fb = unpack_bf16x2(wb[k]);
        acc = fmaf(fa.x, fb.x, acc);
        acc = fmaf(fa.y, fb.y, acc);
        o[k] = pack_bf16x2(p * fa.x, p * fa.y);
      }
      w[u] = make_uint4(o[0], o[1], o[2], o[3]);
    }
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      if (k >= nd) break;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nv) {
          if (mc) st_mc_v4(dsts[k] + (size_t)v * 8, w[u]);
          else st_v4(dsts[k] + (size_t)v * 8, w[u]);
        }
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) dp[it] = acc;
  }
  __threadfence_system();
}

// zero rows for the empty slots (c >= count[e]) of slices [t_lo, t_hi) in the peers' windows
__global__ void __launch_bounds__(WARPS * 32)
    zero_empty_peer_kernel(const int32_t* __restrict__ count, SlotSpace ss, int t_lo, int64_t rows,
                           PeerDst pd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t per_slice = (int64_t)ss.E * ss.Cs;
  const int tt = t_lo + (int)(r / per_slice);
  const int64_t rem = r % per_slice;
  const int e = (int)(rem / ss.Cs);
  const int64_t cs = rem % ss.Cs;
  if ((int64_t)tt * ss.Cs + cs < count[e]) return;
  bf16* dsts[8];
  bool mc;
  const int nd = row_dsts(pd, tt, e, cs, ss, dsts, &mc);
  for (int k = 0; k < nd; ++k)
    for (int v = lane; v < ss.H / 8; v += 32) {
      if (mc) st_mc_v4(dsts[k] + (size_t)v * 8, make_uint4(0, 0, 0, 0));
      else st_v4(dsts[k] + (size_t)v * 8, make_uint4(0, 0, 0, 0));
    }
  __threadfence_system();
}

// ---------------------------------------------------------------- split variants (G_t = 1)
// Rows of this rank's own experts go straight into its expert-space window
// ([E_l][G_ep][C] rows, source block = me); rows of remote experts go to a dense
// slot-space staging buffer, from which the copy engines move them to the peers
// (exchange_ce_dispatch) while the expert GEMM runs on the local block.
__device__ __forceinline__ bf16* split_row(const SplitDst& sd, const SlotSpace& ss, int e, int64_t c) {
  const int owner = e / sd.El;
  if (owner == sd.me)
    return static_cast<bf16*>(sd.loc) + (((size_t)(e - owner * sd.El) * sd.Gep + sd.me) * ss.C + c) * ss.H;
  return static_cast<bf16*>(sd.stage) + ((size_t)e * ss.C + c) * ss.H;
}

__global__ void __launch_bounds__(WARPS * 32)
    dispatch_split_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ tok_of,
                          const int32_t* __restrict__ count, SlotSpace ss, int64_t rows, SplitDst sd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int e = (int)(r / ss.C);
  const int64_t c = r % ss.C;
  bf16* dst = split_row(sd, ss, e, c);
  const int nv = ss.H / 8;
  if (c < count[e]) copy_row<false>(x + (size_t)(tok_of[(size_t)e * ss.C + c] / ss.K) * ss.H, dst, nv, lane);
  else copy_row<true>(nullptr, dst, nv, lane);
}

constexpr int SPLIT_ZW = 4;  // warps per expert zeroing its empty slot rows (combine_bwd_split)
__global__ void __launch_bounds__(WARPS * 32)
    combine_bwd_split_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ O,
                             const int32_t* __restrict__ expert, const int32_t* __restrict__ slot,
                             const float* __restrict__ prob, SlotSpace ss, int64_t T,
                             float* __restrict__ dp, SplitDst sd, const int32_t* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t >= T) {
    // trailing warps, SPLIT_ZW per expert: zero the empty slot rows [count_e, C)
    const int64_t w = t - T;
    if (w >= (int64_t)ss.E * SPLIT_ZW) return;
    const int e = (int)(w / SPLIT_ZW), part = (int)(w % SPLIT_ZW);
    for (int64_t c = count[e] + part; c < ss.C; c += SPLIT_ZW)
      copy_row<true>(nullptr, split_row(sd, ss, e, c), ss.H / 8, lane);
    return;
  }
  for (int kc = 0; kc < ss.K; ++kc) {
    const int64_t it = t * ss.K + kc;
    const int s = slot[it];
    if (s < 0) {
      if (lane == 0) dp[it] = 0.f;
      continue;
    }
    const int e = expert[it];
    const float p = prob[it];
    const bf16* dyr = dy + (size_t)t * ss.H;
    const bf16* orow = O + slot_row(ss, e, s);
    bf16* dst = split_row(sd, ss, e, s);
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
        if (v < nv) st_v4(dst + (size_t)v * 8, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) dp[it] = acc;
  }
}


inline unsigned blocks_for(int64_t n) { return (unsigned)((n + WARPS - 1) / WARPS); }

}  // namespace

cudaError_t dispatch(const void* x, const int32_t* tok_of, const int32_t* count,
                     const SlotSpace& ss, int t_lo, int t_hi, void* D, const int32_t* slot, int64_t T,
                     void* y_zero, cudaStream_t s) {
  const int64_t rows = (int64_t)(t_hi - t_lo) * ss.E * ss.Cs;
  const int64_t zw = y_zero ? (T + 31) / 32 : 0;
  if (rows + zw <= 0) return cudaSuccess;
  dispatch_kernel<<<blocks_for(rows + zw), WARPS * 32, 0, s>>>(static_cast<const bf16*>(x), tok_of,
                                                                count, ss, t_lo, rows,
                                                                static_cast<bf16*>(D), slot, T,
                                                                static_cast<bf16*>(y_zero));
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


cudaError_t dispatch_peer(const void* x, const int32_t* tok_of, const int32_t* count,
                          const SlotSpace& ss, int t_lo, int t_hi, const PeerDst& pd,
                          cudaStream_t s) {
  const int64_t rows = (int64_t)(t_hi - t_lo) * ss.E * ss.Cs;
  if (rows <= 0) return cudaSuccess;
  dispatch_peer_kernel<<<blocks_for(rows), WARPS * 32, 0, s>>>(static_cast<const bf16*>(x), tok_of,
                                                                count, ss, t_lo, rows, pd);
  return cudaGetLastError();
}

cudaError_t combine_bwd_peer(const void* dy, const void* O, const int32_t* expert,
                             const int32_t* slot, const float* prob, const int32_t* count,
                             const int32_t* tok_of, const SlotSpace& ss, int64_t T, int t_lo,
                             int t_hi, float* dp, const PeerDst& pd, cudaStream_t s) {
  (void)tok_of;
  if (T > 0)
    combine_bwd_peer_kernel<<<blocks_for(T), WARPS * 32, 0, s>>>(
        static_cast<const bf16*>(dy), static_cast<const bf16*>(O), expert, slot, prob, ss, T, t_lo,
        t_hi, dp, pd);
  const int64_t rows = (int64_t)(t_hi - t_lo) * ss.E * ss.Cs;
  if (rows > 0)
    zero_empty_peer_kernel<<<blocks_for(rows), WARPS * 32, 0, s>>>(count, ss, t_lo, rows, pd);
  return cudaGetLastError();
}

cudaError_t dispatch_split(const void* x, const int32_t* tok_of, const int32_t* count,
                           const SlotSpace& ss, const SplitDst& sd, cudaStream_t s) {
  const int64_t rows = (int64_t)ss.E * ss.C;
  if (rows <= 0) return cudaSuccess;
  dispatch_split_kernel<<<blocks_for(rows), WARPS * 32, 0, s>>>(static_cast<const bf16*>(x), tok_of, count,
                                                                 ss, rows, sd);
  return cudaGetLastError();
}

cudaError_t combine_bwd_split(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                              const float* prob, const int32_t* count, const SlotSpace& ss, int64_t T,
                              float* dp, const SplitDst& sd, cudaStream_t s) {
  // one launch: a warp per token (dp, dO rows of the kept choices) and SPLIT_ZW warps per
  // expert zeroing its empty slot rows
  const int64_t warps = T + (int64_t)ss.E * SPLIT_ZW;
  if (warps > 0 && ss.C > 0)
    combine_bwd_split_kernel<<<blocks_for(warps), WARPS * 32, 0, s>>>(
        static_cast<const bf16*>(dy), static_cast<const bf16*>(O), expert, slot, prob, ss, T, dp, sd, count);
  return cudaGetLastError();
}

}  // namespace moe
