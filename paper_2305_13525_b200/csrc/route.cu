// route.cu — F1 (top-1 gate) and F2 (capacity slot scan), SURVEY §8(a).
//
// F1 gate: l = x Wg with fp32 accumulation, softmax max/denominator, lowest-index
// argmax, top-2 gap, p = softmax(l)[e*] (R1, R4). One warp owns TPW
// tokens at a time; lane l handles h = 8 l + 256 i + j, so each lane loads one
// 16-byte vector of x per 256-wide H step (fully coalesced), and the matching
// Wg values come from a shared-memory copy laid out so the two LDS.128 per
// (e, i) are conflict-free across the warp. Partial sums per lane cover H/32
// terms, then a butterfly reduce: a tree summation whose error (~1e-7 on N(0,1)
// logits) stays well below the 1e-6 tie threshold of BASELINE.json.
//
// F2 slots: slot_t = #{t' < t : e*(t') = e*(t)} (R3), in two passes over
// 1024-token blocks: (a) per-block warp-match ranks + block histogram,
// (b) block prefix per expert, slot/keep decision, count[E], and the inverse
// map tok_of[e][slot] used by the slot-parallel dispatch.
#include <float.h>

#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int GATE_WARPS = 8;
constexpr int HC = 256;  // H chunk staged in shared memory per pass

template <int EMAX, int TPW>
__global__ void __launch_bounds__(GATE_WARPS * 32)
    gate_kernel(const bf16* __restrict__ x, const float* __restrict__ wg,
                const int32_t* __restrict__ forced, int64_t T, int H, int E,
                float* __restrict__ logits, int32_t* __restrict__ expert,
                float* __restrict__ prob, float* __restrict__ gap, int32_t* __restrict__ ties) {
  // ws[e][HC] permuted: h_local = 8 l + 4 half + q  ->  e*HC + half*128 + l*4 + q
  extern __shared__ __align__(16) float ws[];  // [EMAX * HC]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tok0 = ((int64_t)blockIdx.x * GATE_WARPS + warp) * TPW;

  float acc[TPW][EMAX];
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[t][e] = 0.f;

  for (int h0 = 0; h0 < H; h0 += HC) {
    __syncthreads();
    for (int i = threadIdx.x; i < EMAX * HC; i += blockDim.x) {
      const int e = i / HC, hl = i % HC;
      const int l = hl >> 3, half = (hl >> 2) & 1, q = hl & 3;
      const int h = h0 + hl;
      ws[e * HC + half * 128 + l * 4 + q] = (e < E && h < H) ? wg[(size_t)h * E + e] : 0.f;
    }
    __syncthreads();
    const int h = h0 + 8 * lane;
    if (h < H) {
      float xv[TPW][8];
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int64_t tok = tok0 + t;
        uint4 u = make_uint4(0, 0, 0, 0);
        if (tok < T) u = ld_nc_v4(x + (size_t)tok * H + h);
        float2 f0 = unpack_bf16x2(u.x), f1 = unpack_bf16x2(u.y), f2 = unpack_bf16x2(u.z),
               f3 = unpack_bf16x2(u.w);
        xv[t][0] = f0.x; xv[t][1] = f0.y; xv[t][2] = f1.x; xv[t][3] = f1.y;
        xv[t][4] = f2.x; xv[t][5] = f2.y; xv[t][6] = f3.x; xv[t][7] = f3.y;
      }
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        const float4 w0 = *reinterpret_cast<const float4*>(&ws[e * HC + lane * 4]);
        const float4 w1 = *reinterpret_cast<const float4*>(&ws[e * HC + 128 + lane * 4]);
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          float a = acc[t][e];
          a = fmaf(xv[t][0], w0.x, a); a = fmaf(xv[t][1], w0.y, a);
          a = fmaf(xv[t][2], w0.z, a); a = fmaf(xv[t][3], w0.w, a);
          a = fmaf(xv[t][4], w1.x, a); a = fmaf(xv[t][5], w1.y, a);
          a = fmaf(xv[t][6], w1.z, a); a = fmaf(xv[t][7], w1.w, a);
          acc[t][e] = a;
        }
      }
    }
  }
  // butterfly reduction of the 32 lane partials (fixed tree order)
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[t][e] = warp_sum(acc[t][e]);

  if (lane < TPW) {
    // every lane holds every sum; lane t finalises token tok0 + t
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      if (t != lane) continue;
      const int64_t tok = tok0 + t;
      if (tok >= T) continue;
      float m = -FLT_MAX, m2 = -FLT_MAX;
      int best = 0;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        const float v = acc[t][e];
        logits[(size_t)tok * E + e] = v;
        if (v > m) { m2 = m; m = v; best = e; }
        else if (v > m2) { m2 = v; }
      }
      float den = 0.f;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        den += expf(acc[t][e] - m);
      }
      int chosen = best;
      if (forced) chosen = forced[tok];
      float lc = m;
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e == chosen) lc = acc[t][e];
      const float g = (E > 1) ? (m - m2) : FLT_MAX;
      expert[tok] = chosen;
      prob[tok] = expf(lc - m) / den;
      gap[tok] = g;
      if (g < 1e-6f) atomicAdd(ties, 1);
    }
  }
}

constexpr int SCAN_BLOCK = 1024;

// (a) rank of each token among same-expert tokens of its 1024-block + block histogram.
__global__ void __launch_bounds__(SCAN_BLOCK)
    slot_local_kernel(const int32_t* __restrict__ expert, int64_t T, int E,
                      int32_t* __restrict__ local_rank, int32_t* __restrict__ block_hist) {
  __shared__ int32_t wh[32][65];  // per-warp histogram, E <= 64
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  for (int i = threadIdx.x; i < 32 * 65; i += SCAN_BLOCK) (&wh[0][0])[i] = 0;
  __syncthreads();
  const int e = (t < T) ? expert[t] : -1;
  const uint32_t peers = __match_any_sync(0xffffffffu, e);
  const int rank_in_warp = __popc(peers & ((1u << lane) - 1));
  if (e >= 0 && rank_in_warp == 0) wh[warp][e] = __popc(peers);
  __syncthreads();
  // exclusive scan over warps, per expert (thread e)
  if (threadIdx.x < E) {
    int run = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = wh[w][threadIdx.x];
      wh[w][threadIdx.x] = run;
      run += c;
    }
    block_hist[(size_t)blockIdx.x * E + threadIdx.x] = run;
  }
  __syncthreads();
  if (t < T) local_rank[t] = wh[warp][e] + rank_in_warp;
}

// (b) slot = block prefix + local rank; keep iff slot < C; inverse map; counts.
__global__ void __launch_bounds__(SCAN_BLOCK)
    slot_final_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ local_rank,
                      const int32_t* __restrict__ block_hist, int64_t T, int E, int64_t C,
                      int nblocks, int32_t* __restrict__ slot, int32_t* __restrict__ tok_of,
                      int32_t* __restrict__ count, int32_t* __restrict__ load) {
  __shared__ int32_t prefix[64];
  if (threadIdx.x < E) {
    int run = 0, total = 0;
    for (int b = 0; b < nblocks; ++b) {
      const int c = block_hist[(size_t)b * E + threadIdx.x];
      if (b < (int)blockIdx.x) run += c;
      total += c;
    }
    prefix[threadIdx.x] = run;
    if (blockIdx.x == 0) {
      load[threadIdx.x] = total;
      count[threadIdx.x] = (int)((int64_t)total < C ? total : C);
    }
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  if (t >= T) return;
  const int e = expert[t];
  const int64_t s = (int64_t)prefix[e] + local_rank[t];
  if (s < C) {
    slot[t] = (int32_t)s;
    tok_of[(size_t)e * C + s] = (int32_t)t;
  } else {
    slot[t] = -1;
  }
}

template <int EMAX, int TPW>
cudaError_t launch_gate(const RouteArgs& a, cudaStream_t s) {
  const int64_t per_cta = (int64_t)GATE_WARPS * TPW;
  const int64_t grid = (a.T + per_cta - 1) / per_cta;
  const int smem = EMAX * HC * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<EMAX, TPW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gate_kernel<EMAX, TPW><<<(unsigned)grid, GATE_WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(a.x), a.wg, a.forced, a.T, a.H, a.E, a.logits, a.expert, a.prob,
      a.gap, a.ties);
  return cudaGetLastError();
}

}  // namespace

cudaError_t route(const RouteArgs& a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(a.ties, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  if (a.T == 0) {
    e = cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.E, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.load, 0, sizeof(int32_t) * a.E, s);
    return e;
  }
  if (a.E <= 4) e = launch_gate<4, 8>(a, s);
  else if (a.E <= 8) e = launch_gate<8, 8>(a, s);
  else if (a.E <= 16) e = launch_gate<16, 4>(a, s);
  else if (a.E <= 32) e = launch_gate<32, 2>(a, s);
  else e = launch_gate<64, 1>(a, s);
  if (e != cudaSuccess) return e;
  const int nblocks = (int)((a.T + SCAN_BLOCK - 1) / SCAN_BLOCK);
  slot_local_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.T, a.E, a.local_rank, a.block_hist);
  slot_final_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.local_rank, a.block_hist, a.T, a.E,
                                                   a.C, nblocks, a.slot, a.tok_of, a.count, a.load);
  return cudaGetLastError();
}

}  // namespace moe
