// route.cu — F1 (top-1 gate) and F2 (capacity slot scan), SURVEY §8(a).
//
// F1 gate: l = x Wg with fp32 accumulation, softmax max/denominator, lowest-index
// argmax, top-2 gap, p = softmax(l)[e*] (R1, R4). The contraction is
// ALU-bound on CUDA cores (E flop/byte): Wg sits in shared memory
// (resident when H*E*4 <= 128 KiB, else streamed per H-chunk), each 128 B Wg line
// feeds 4 tokens by broadcast, and the FMAs are packed fma.rn.f32x2. Every lane
// sums H/8 terms in two (even/odd) chains and the 8 lanes of a token are combined
// by a fixed xor tree: error ~1e-7 on N(0,1) logits, well below the 1e-6 tie
// threshold of BASELINE.json.
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


// One CTA = GATE_WARPS warps; a warp = 4 token groups (q = lane / 8) of 8 lanes (l8) that
// split H: lane l8 owns h = 64 blk + 8 l8 + [0, 8) of every 64-wide step. Each
// lane carries TPW tokens (token = base + 4 i + q), so a warp holds 4*TPW tokens.
// Accumulators are float2 (even h, odd h) updated with fma.rn.f32x2; the final
// sum is (even + odd) then a 3-level xor-shuffle over the 8 lanes.
template <int EMAX, int TPW, int GATE_WARPS>
__global__ void __launch_bounds__(GATE_WARPS * 32, 1)
    gate_kernel(const bf16* __restrict__ x, const float* __restrict__ wg,
                const int32_t* __restrict__ forced, int64_t T, int H, int E, int hch,
                float* __restrict__ logits, int32_t* __restrict__ expert,
                float* __restrict__ prob, float* __restrict__ gap, int32_t* __restrict__ ties) {
  extern __shared__ __align__(16) float ws[];  // [EMAX][hch], see ws_index
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane >> 3, l8 = lane & 7;
  constexpr int PER_WARP = 4 * TPW;
  constexpr int PER_CTA = GATE_WARPS * PER_WARP;
  constexpr int PD = EMAX >= 64 ? 2 : 4;  // x prefetch depth (64-wide H steps)
  const int nchunks = (H + hch - 1) / hch;
  const bool resident = nchunks == 1;
  if (resident) {
    stage_wg(ws, wg, 0, hch, H, E);
    __syncthreads();
  }
  const int64_t nbatch = (T + PER_CTA - 1) / PER_CTA;
  for (int64_t b = blockIdx.x; b < nbatch; b += gridDim.x) {
    const int64_t base = b * PER_CTA + warp * PER_WARP + q;
    float2 acc[TPW][EMAX];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int e = 0; e < EMAX; ++e) acc[i][e] = make_float2(0.f, 0.f);

    for (int c = 0; c < nchunks; ++c) {
      const int h0 = c * hch;
      if (!resident) {
        __syncthreads();
        stage_wg(ws, wg, h0, hch, H, E);
        __syncthreads();
      }
      const int nblk = (H - h0 < hch ? H - h0 : hch) >> 6;
      // software pipeline: x for steps blk .. blk+PD-1 in flight (PD*TPW 16-byte loads per lane)
      uint4 buf[PD][TPW];
#pragma unroll
      for (int s = 0; s < PD; ++s)
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int64_t tok = base + 4 * i;
          buf[s][i] = (tok < T && s < nblk) ? ld_nc_v4(x + (size_t)tok * H + h0 + 64 * s + 8 * l8)
                                            : make_uint4(0, 0, 0, 0);
        }
      for (int blk0 = 0; blk0 < nblk; blk0 += PD) {
#pragma unroll
        for (int s = 0; s < PD; ++s) {
          const int blk = blk0 + s;
          if (blk < nblk) {
            float2 xv[TPW][4];
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
              xv[i][0] = unpack_bf16x2(buf[s][i].x); xv[i][1] = unpack_bf16x2(buf[s][i].y);
              xv[i][2] = unpack_bf16x2(buf[s][i].z); xv[i][3] = unpack_bf16x2(buf[s][i].w);
              const int64_t tok = base + 4 * i;
              if (tok < T && blk + PD < nblk)
                buf[s][i] = ld_nc_v4(x + (size_t)tok * H + h0 + 64 * (blk + PD) + 8 * l8);
            }
            const float* wrow = ws + blk * 64 + l8 * 4;
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
              const float4 w0 = *reinterpret_cast<const float4*>(wrow + e * hch);
              const float4 w1 = *reinterpret_cast<const float4*>(wrow + e * hch + 32);
              const float2 p0 = make_float2(w0.x, w0.y), p1 = make_float2(w0.z, w0.w);
              const float2 p2 = make_float2(w1.x, w1.y), p3 = make_float2(w1.z, w1.w);
#pragma unroll
              for (int i = 0; i < TPW; ++i) {
                ffma2(acc[i][e], xv[i][0], p0);
                ffma2(acc[i][e], xv[i][1], p1);
                ffma2(acc[i][e], xv[i][2], p2);
                ffma2(acc[i][e], xv[i][3], p3);
              }
            }
          }
        }
      }
    }
    // (even + odd), then tree over the 8 lanes of the token group (result in .x)
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        float v = acc[i][e].x + acc[i][e].y;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        acc[i][e].x = v;
      }
    // lane l8 == i finalises token base + 4 i
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t tok = base + 4 * i;
      if (l8 != i || tok >= T) continue;
      float m = -FLT_MAX, m2 = -FLT_MAX;
      int best = 0;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        const float v = acc[i][e].x;
        logits[(size_t)tok * E + e] = v;
        if (v > m) { m2 = m; m = v; best = e; }
        else if (v > m2) { m2 = v; }
      }
      float den = 0.f;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        den += expf(acc[i][e].x - m);
      }
      const int chosen = forced ? forced[tok] : best;
      float lc = m;
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e == chosen) lc = acc[i][e].x;
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

int g_sms = 0;

template <int EMAX, int TPW, int GATE_WARPS>
cudaError_t launch_gate(const RouteArgs& a, cudaStream_t s) {
  constexpr int hmax = wg_chunk(EMAX);
  const int hch = a.H < hmax ? a.H : hmax;
  const int smem = EMAX * hch * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<EMAX, TPW, GATE_WARPS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t per_cta = (int64_t)GATE_WARPS * 4 * TPW;
  int64_t grid = (a.T + per_cta - 1) / per_cta;
  if (hch >= a.H && grid > g_sms) grid = g_sms;  // Wg resident: persistent over token batches
  gate_kernel<EMAX, TPW, GATE_WARPS><<<(unsigned)grid, GATE_WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(a.x), a.wg, a.forced, a.T, a.H, a.E, hch, a.logits, a.expert,
      a.prob, a.gap, a.ties);
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
  if (a.E <= 4) e = launch_gate<4, 2, 16>(a, s);
  else if (a.E <= 8) e = launch_gate<8, 2, 16>(a, s);
  else if (a.E <= 16) e = launch_gate<16, 1, 16>(a, s);
  else if (a.E <= 32) e = launch_gate<32, 1, 16>(a, s);
  else e = launch_gate<64, 1, 8>(a, s);
  if (e != cudaSuccess) return e;
  const int nblocks = (int)((a.T + SCAN_BLOCK - 1) / SCAN_BLOCK);
  slot_local_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.T, a.E, a.local_rank, a.block_hist);
  slot_final_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.local_rank, a.block_hist, a.T, a.E,
                                                   a.C, nblocks, a.slot, a.tok_of, a.count, a.load);
  return cudaGetLastError();
}

}  // namespace moe
