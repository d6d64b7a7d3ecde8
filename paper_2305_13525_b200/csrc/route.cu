// route.cu — F1 (top-1 gate) and F2 (capacity slot scan), SURVEY §8(a).
//
// F1 gate: l = x Wg with fp32 accumulation, softmax max/denominator, lowest-index
// argmax, top-2 gap, p = softmax(l)[e*] (R1, R4). The contraction is
// ALU-bound on CUDA cores (E flop/byte): Wg sits in shared memory
// (resident when H*E*4 <= 128 KiB, else streamed per H-chunk) and each Wg value
// loaded by a lane feeds TPW tokens from registers (an LDS.128 costs 4 wavefronts
// whatever the address pattern, so reuse per lane is what bounds shared-memory
// traffic). Every lane sums H/32 terms, then a fixed butterfly over the warp:
// error ~1e-7 on N(0,1) logits, well below the 1e-6 tie threshold of BASELINE.json.
//
// F2 slots: slot_t = #{t' < t : e*(t') = e*(t)} (R3), in two passes over
// 1024-token blocks: (a) per-block warp-match ranks + block histogram,
// (b) block prefix per expert, slot/keep decision, count[E], and the inverse
// map tok_of[e][slot] used by the slot-parallel dispatch.
#include <atomic>
#include <float.h>

#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {


// Wg staged as expert pairs: wp[ep][blk][kp][lane][4] holds, for h = 256 blk + 8 lane
// + 2 kp + {0,1} and e = 2 ep + {0,1}: (w[h][e0], w[h][e1], w[h+1][e0], w[h+1][e1]).
// One LDS.128 per (ep, blk, kp) across the warp reads 512 contiguous bytes.
__device__ __forceinline__ int wp_index(int e, int hl, int hch) {
  const int blk = hl >> 8, r = hl & 255, ln = r >> 3, k = r & 7;
  return (e >> 1) * (2 * hch) + blk * 512 + (k >> 1) * 128 + ln * 4 + (k & 1) * 2 + (e & 1);
}

__device__ __forceinline__ void stage_wg_pairs(float* ws, const float* __restrict__ wg, int h0,
                                               int hch, int H, int E, int emax, int e0) {
  constexpr int U = 16;
  const int n = hch * emax;
  const int nt = blockDim.x;
  for (int b = threadIdx.x; b < n; b += U * nt) {
    float v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = b + k * nt;
      const int hl = i / emax, e = i - hl * emax;
      v[k] = (i < n && e0 + e < E && h0 + hl < H) ? __ldg(wg + (size_t)(h0 + hl) * E + e0 + e) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = b + k * nt;
      if (i < n) {
        const int hl = i / emax, e = i - hl * emax;
        ws[wp_index(e, hl, hch)] = v[k];
      }
    }
  }
}

// Routing decision of one token from its E logits (R1, R4, R5; top-2: R22).
template <int EMAX>
__device__ __forceinline__ void finalize_token(const float (&lv)[EMAX], int64_t tok, int E, int K,
                                               const int32_t* __restrict__ forced,
                                               int32_t* __restrict__ expert, float* __restrict__ prob,
                                               float* __restrict__ gap, int32_t* __restrict__ ties) {
  float m = -FLT_MAX, m2 = -FLT_MAX;
  int best = 0;
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    if (e >= E) break;
    const float v = lv[e];
    if (v > m) { m2 = m; m = v; best = e; }
    else if (v > m2) { m2 = v; }
  }
  float den = 0.f;
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    if (e >= E) break;
    den += expf(lv[e] - m);
  }
  if (K == 2) {  // R22: second = lowest-index max over e != best; gap over the top 3
    float v2 = -FLT_MAX, v3 = -FLT_MAX;
    int e2 = best == 0 ? 1 : 0;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      if (e >= E) break;
      if (e == best) continue;
      const float v = lv[e];
      if (v > v2) { v3 = v2; v2 = v; e2 = e; }
      else if (v > v3) { v3 = v; }
    }
    const float g = E > 2 ? fminf(m - v2, v2 - v3) : m - v2;
    const float s1 = 1.f / den, s2 = expf(v2 - m) / den;
    expert[2 * tok] = best;
    expert[2 * tok + 1] = e2;
    prob[2 * tok] = s1 / (s1 + s2);
    prob[2 * tok + 1] = s2 / (s1 + s2);
    gap[tok] = g;
    if (g < 1e-6f) atomicAdd(ties, 1);
    return;
  }
  const int chosen = forced ? forced[tok] : best;
  float lc = m;
#pragma unroll
  for (int e = 0; e < EMAX; ++e)
    if (e == chosen) lc = lv[e];
  const float g = (E > 1) ? (m - m2) : FLT_MAX;
  expert[tok] = chosen;
  prob[tok] = expf(lc - m) / den;
  gap[tok] = g;
  if (g < 1e-6f) atomicAdd(ties, 1);
}

// Expert-split gate, second pass: one thread per token reads its E logits (written by
// the logits-only passes) and takes the same routing decision.
template <int EMAX>
__global__ void __launch_bounds__(256)
    gate_finalize_kernel(const float* __restrict__ logits, const int32_t* __restrict__ forced, int64_t T,
                         int E, int K, int32_t* __restrict__ expert, float* __restrict__ prob,
                         float* __restrict__ gap, int32_t* __restrict__ ties) {
  const int64_t tok = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tok >= T) return;
  float lv[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) lv[e] = e < E ? logits[(size_t)tok * E + e] : -FLT_MAX;
  finalize_token<EMAX>(lv, tok, E, K, forced, expert, prob, gap, ties);
}

// One warp owns TPW tokens at a time; lane l covers h = 256 i + 8 l + [0, 8).
// x streams through a per-warp double buffer in shared memory (cp.async, one
// coalesced 16-byte piece per lane per token per 256-wide step); Wg comes from
// shared memory (resident when it fits in 128 KiB, else streamed per H-chunk);
// every Wg pair a lane loads is reused for its TPW tokens, and the FMAs are packed
// fma.rn.f32x2 over expert pairs: (acc_e0, acc_e1) += (x, x) * (w_e0, w_e1).
// Each lane sums H/32 terms per expert in h order, then a fixed butterfly.
template <int EMAX, int TPW, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    gate_kernel(const bf16* __restrict__ x, const float* __restrict__ wg,
                const int32_t* __restrict__ forced, int64_t T, int H, int E, int hch, int K,
                bool logits_only,
                float* __restrict__ logits, int32_t* __restrict__ expert,
                float* __restrict__ prob, float* __restrict__ gap, int32_t* __restrict__ ties) {
  constexpr int EP = EMAX / 2;
  // expert-split pass (logits_only): CTA row blockIdx.y covers experts [e0, e0 + EMAX)
  const int e0 = logits_only ? (int)blockIdx.y * EMAX : 0;
  extern __shared__ __align__(16) float ws[];  // [EP][2*hch] (see wp_index), then x buffers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // x double buffer of this warp: [2][TPW][256] bf16
  bf16* xs = reinterpret_cast<bf16*>(ws + EMAX * hch) + (size_t)warp * 2 * TPW * 256;
  constexpr int PER_CTA = WARPS * TPW;
  const int nchunks = (H + hch - 1) / hch;
  const bool resident = nchunks == 1;
  if (resident) {
    stage_wg_pairs(ws, wg, 0, hch, H, E, EMAX, e0);
    __syncthreads();
  }
  const int64_t nbatch = (T + PER_CTA - 1) / PER_CTA;
  for (int64_t b = blockIdx.x; b < nbatch; b += gridDim.x) {
    const int64_t tok0 = b * PER_CTA + warp * TPW;
    float2 acc[TPW][EP];
#pragma unroll
    for (int t = 0; t < TPW; ++t)
#pragma unroll
      for (int e = 0; e < EP; ++e) acc[t][e] = make_float2(0.f, 0.f);

    for (int c = 0; c < nchunks; ++c) {
      const int h0 = c * hch;
      if (!resident) {
        __syncthreads();
        stage_wg_pairs(ws, wg, h0, hch, H, E, EMAX, e0);
        __syncthreads();
      }
      const int hlen = H - h0 < hch ? H - h0 : hch;
      const int nblk = (hlen + 255) >> 8;
      auto issue = [&](int blk) {
        bf16* dst = xs + (blk & 1) * TPW * 256;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int h = 256 * blk + 8 * lane;
          const int64_t tok = tok0 + t;
          const bool ok = blk < nblk && h < hlen && tok < T;
          cp_async_16(smem_u32(dst + t * 256 + 8 * lane), ok ? x + (size_t)tok * H + h0 + h : x, ok);
        }
        cp_async_commit();
      };
      issue(0);
      for (int blk = 0; blk < nblk; ++blk) {
        issue(blk + 1);
        cp_async_wait_1();  // this lane's pieces of step blk have landed
        const bf16* cur = xs + (blk & 1) * TPW * 256;
        uint4 xv[TPW];
#pragma unroll
        for (int t = 0; t < TPW; ++t)
          xv[t] = *reinterpret_cast<const uint4*>(cur + t * 256 + 8 * lane);
        const float* wrow = ws + blk * 512 + lane * 4;
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          float2 xd0[TPW], xd1[TPW];  // (x, x) for h = 2 kp and 2 kp + 1
#pragma unroll
          for (int t = 0; t < TPW; ++t) {
            const uint32_t u = kp == 0 ? xv[t].x : kp == 1 ? xv[t].y : kp == 2 ? xv[t].z : xv[t].w;
            const float2 f = unpack_bf16x2(u);
            xd0[t] = make_float2(f.x, f.x);
            xd1[t] = make_float2(f.y, f.y);
          }
#pragma unroll
          for (int ep = 0; ep < EP; ++ep) {
            const float4 w = *reinterpret_cast<const float4*>(wrow + ep * 2 * hch + kp * 128);
            const float2 w0 = make_float2(w.x, w.y), w1 = make_float2(w.z, w.w);
#pragma unroll
            for (int t = 0; t < TPW; ++t) {
              ffma2(acc[t][ep], xd0[t], w0);
              ffma2(acc[t][ep], xd1[t], w1);
            }
          }
        }
      }
      cp_async_wait_0();
    }
    // fixed butterfly over the 32 lanes (every lane ends with every sum)
#pragma unroll
    for (int t = 0; t < TPW; ++t)
#pragma unroll
      for (int ep = 0; ep < EP; ++ep) {
        acc[t][ep].x = warp_sum(acc[t][ep].x);
        acc[t][ep].y = warp_sum(acc[t][ep].y);
      }
    // lane t finalises token tok0 + t
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int64_t tok = tok0 + t;
      if (lane != t || tok >= T) continue;
      float lv[EMAX];
#pragma unroll
      for (int ep = 0; ep < EP; ++ep) {
        lv[2 * ep] = acc[t][ep].x;
        lv[2 * ep + 1] = acc[t][ep].y;
      }
      if (logits_only) {  // expert-split pass: this CTA's EMAX experts starting at e0
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
          if (e0 + e < E) logits[(size_t)tok * E + e0 + e] = lv[e];
        continue;
      }
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e < E) logits[(size_t)tok * E + e] = lv[e];
      finalize_token<EMAX>(lv, tok, E, K, forced, expert, prob, gap, ties);
    }
  }
}

constexpr int SCAN_BLOCK = 1024;

// ---------------------------------------------------------------- random priority (R20)
// sigma(i): token at priority position i. 4-round Feistel network on 2m bits (the
// smallest 4^m >= T), cycle-walked into [0, T): a bijection of [0, T). Same
// construction as oracle.priority_order (counter-based; both sides implement it).
struct Prio {
  int on, m;
  uint32_t mask, k[4];
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t feistel(uint32_t x, const Prio& p) {
  uint32_t L = x >> p.m, R = x & p.mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t nl = R;
    R = L ^ (mix32(R ^ p.k[r]) & p.mask);
    L = nl;
  }
  return (L << p.m) | R;
}

__device__ __forceinline__ int64_t prio_token(int64_t i, int64_t T, const Prio& p) {
  if (!p.on) return i;
  uint32_t x = feistel((uint32_t)i, p);
  while ((int64_t)x >= T) x = feistel(x, p);
  return x;
}

// Scan items i in [0, K*T): pass k = i / T (first choices, then second choices, R22),
// priority position q = i % T -> token prio_token(q); the item id t*K + k indexes the
// per-(token, choice) arrays.
__device__ __forceinline__ int64_t item_id(int64_t i, int64_t T, int K, const Prio& p) {
  const int64_t k = K == 1 ? 0 : i / T;
  return prio_token(i - k * T, T, p) * K + k;
}

// (a) rank of each item among same-expert items of its 1024-block + block histogram.
// Positions i = priority order (token order unless random priority is on).
__global__ void __launch_bounds__(SCAN_BLOCK)
    slot_local_kernel(const int32_t* __restrict__ expert, int64_t T, int K, int E, Prio pr,
                      int32_t* __restrict__ local_rank, int32_t* __restrict__ block_hist) {
  const int64_t N = T * K;
  __shared__ int32_t wh[32][65];  // per-warp histogram, E <= 64
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;
  for (int i = threadIdx.x; i < 32 * 65; i += SCAN_BLOCK) (&wh[0][0])[i] = 0;
  __syncthreads();
  const int e = (t < N) ? expert[item_id(t, T, K, pr)] : -1;
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
  if (t < N) local_rank[t] = wh[warp][e] + rank_in_warp;
}

// (b) slot = block prefix + local rank; keep iff slot < C; inverse map; counts.
__global__ void __launch_bounds__(SCAN_BLOCK)
    slot_final_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ local_rank,
                      const int32_t* __restrict__ block_hist, int64_t T, int K, int E, int64_t C,
                      int nblocks, Prio pr, int32_t* __restrict__ slot, int32_t* __restrict__ tok_of,
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
  const int64_t i = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x;  // scan item
  if (i >= T * K) return;
  const int64_t it = item_id(i, T, K, pr);
  const int e = expert[it];
  const int64_t s = (int64_t)prefix[e] + local_rank[i];
  if (s < C) {
    slot[it] = (int32_t)s;
    tok_of[(size_t)e * C + s] = (int32_t)it;  // item id: token * K + choice
  } else {
    slot[it] = -1;
  }
}

// ---------------------------------------------------------------- aux loss (R21)
// P_e = (1/T) sum_t softmax(l_t)_e: AUX_GRID CTAs over fixed token ranges, each
// thread sums its tokens in order, then a fixed butterfly per warp and warps in
// order: deterministic. aux_final: f_e = load_e / T, l_aux = coef E sum_e f_e P_e.
template <int EMAX>
__global__ void __launch_bounds__(256)
    aux_partial_kernel(const float* __restrict__ logits, const int32_t* __restrict__ expert, int64_t T,
                       int K, int E, float* __restrict__ partial) {
  __shared__ float ws[8][EMAX];
  __shared__ int wc[8][EMAX];
  int cnt[EMAX];  // first choices (f_e counts only the first choice, R21/R22)
#pragma unroll
  for (int e = 0; e < EMAX; ++e) cnt[e] = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (T + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t t1 = t0 + per < T ? t0 + per : T;
  float acc[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) acc[e] = 0.f;
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    float l[EMAX];
    float m = -FLT_MAX;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      l[e] = e < E ? logits[(size_t)t * E + e] : -FLT_MAX;
      m = fmaxf(m, l[e]);
    }
    float den = 0.f;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      l[e] = e < E ? expf(l[e] - m) : 0.f;
      den += l[e];
    }
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[e] += l[e] / den;
    const int e1 = expert[(size_t)t * K];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) cnt[e] += e == e1;
  }
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    const float v = warp_sum(acc[e]);
    int c = cnt[e];
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) { ws[warp][e] = v; wc[warp][e] = c; }
  }
  __syncthreads();
  if (threadIdx.x < E) {
    float v = 0.f;
    int c = 0;
    for (int w = 0; w < 8; ++w) { v += ws[w][threadIdx.x]; c += wc[w][threadIdx.x]; }
    partial[(size_t)blockIdx.x * E + threadIdx.x] = v;
    reinterpret_cast<int32_t*>(partial + (size_t)AUX_GRID * E)[(size_t)blockIdx.x * E + threadIdx.x] = c;
  }
}

__global__ void aux_final_kernel(const float* __restrict__ partial, int64_t T, int E, float coef,
                                 float* __restrict__ out) {
  __shared__ float fp[64];
  const int e = threadIdx.x;
  if (e < E) {
    float P = 0.f;
    for (int b = 0; b < AUX_GRID; ++b) P += partial[(size_t)b * E + e];
    P /= (float)T;
    int64_t n1 = 0;
    const int32_t* cnt = reinterpret_cast<const int32_t*>(partial + (size_t)AUX_GRID * E);
    for (int b = 0; b < AUX_GRID; ++b) n1 += cnt[(size_t)b * E + e];
    const float f = (float)n1 / (float)T;
    out[e] = f;
    fp[e] = f * P;
  }
  __syncthreads();
  if (e == 0) {
    float sum = 0.f;
    for (int j = 0; j < E; ++j) sum += fp[j];
    out[E] = coef * (float)E * sum;
  }
}

std::atomic<int> g_sms{0};

template <int EMAX, int TPW, int WARPS>
cudaError_t launch_gate(const RouteArgs& a, cudaStream_t s) {
  constexpr int hmax = wg_chunk(EMAX);
  const int hpad = (a.H + 255) & ~255;
  const int hch = hpad < hmax ? hpad : hmax;
  const int smem = EMAX * hch * 4 + WARPS * 2 * TPW * 256 * 2;
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<EMAX, TPW, WARPS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         128 * 1024 + WARPS * 2 * TPW * 256 * 2);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g_sms) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms = n;
  }
  const int64_t per_cta = (int64_t)WARPS * TPW;
  int64_t grid = (a.T + per_cta - 1) / per_cta;
  if (hch >= a.H && grid > g_sms) grid = g_sms;  // Wg resident: persistent over token batches
  gate_kernel<EMAX, TPW, WARPS><<<(unsigned)grid, WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(a.x), a.wg, a.forced, a.T, a.H, a.E, hch, a.K, false, a.logits, a.expert,
      a.prob, a.gap, a.ties);
  return cudaGetLastError();
}

// Expert split (Wg of all E experts does not fit in 128 KiB of shared memory, e.g.
// H = 4096 with E = 16, or H = 2560 with E = 32): groups of EG experts whose [H][EG]
// slice stays resident (<= 160 KiB), one grid row per group, logits only; then
// gate_finalize_kernel takes the routing decision from the full logit rows.
constexpr int SPLIT_WG_BYTES = 160 * 1024;

template <int EG>
cudaError_t launch_gate_split(const RouteArgs& a, int hpad, cudaStream_t s) {
  constexpr int TPW = 4, WARPS = 16;
  const int smem = EG * hpad * 4 + WARPS * 2 * TPW * 256 * 2;
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<EG, TPW, WARPS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SPLIT_WG_BYTES + WARPS * 2 * TPW * 256 * 2);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g_sms) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms = n;
  }
  const int groups = (a.E + EG - 1) / EG;
  const int64_t per_cta = (int64_t)WARPS * TPW;
  int64_t gx = (a.T + per_cta - 1) / per_cta;
  const int64_t cap = (g_sms + groups - 1) / groups;
  if (gx > cap) gx = cap;
  gate_kernel<EG, TPW, WARPS><<<dim3((unsigned)gx, groups), WARPS * 32, smem, s>>>(
      static_cast<const bf16*>(a.x), a.wg, a.forced, a.T, a.H, a.E, hpad, a.K, true, a.logits, a.expert,
      a.prob, a.gap, a.ties);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const unsigned fb = (unsigned)((a.T + 255) / 256);
  if (a.E <= 16) gate_finalize_kernel<16><<<fb, 256, 0, s>>>(a.logits, a.forced, a.T, a.E, a.K, a.expert, a.prob, a.gap, a.ties);
  else if (a.E <= 32) gate_finalize_kernel<32><<<fb, 256, 0, s>>>(a.logits, a.forced, a.T, a.E, a.K, a.expert, a.prob, a.gap, a.ties);
  else gate_finalize_kernel<64><<<fb, 256, 0, s>>>(a.logits, a.forced, a.T, a.E, a.K, a.expert, a.prob, a.gap, a.ties);
  return cudaGetLastError();
}

}  // namespace

cudaError_t route(const RouteArgs& a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(a.ties, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  if (a.T == 0) {
    e = cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.E, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.load, 0, sizeof(int32_t) * a.E, s);
    if (e == cudaSuccess && a.aux_out) e = cudaMemsetAsync(a.aux_out, 0, sizeof(float) * (a.E + 1), s);
    return e;
  }
  const int hpad = (a.H + 255) & ~255;
  const int emax = a.E <= 4 ? 4 : a.E <= 8 ? 8 : a.E <= 16 ? 16 : a.E <= 32 ? 32 : 64;
  const bool resident = (int64_t)emax * hpad * 4 <= 128 * 1024;
  if (!resident && a.E > 4 && (int64_t)16 * hpad * 4 <= SPLIT_WG_BYTES) e = launch_gate_split<16>(a, hpad, s);
  else if (!resident && a.E > 4 && (int64_t)8 * hpad * 4 <= SPLIT_WG_BYTES) e = launch_gate_split<8>(a, hpad, s);
  else if (a.E <= 4) e = launch_gate<4, 4, 16>(a, s);
  else if (a.E <= 8) e = launch_gate<8, 4, 16>(a, s);
  else if (a.E <= 16) e = launch_gate<16, 4, 16>(a, s);
  else if (a.E <= 32) e = launch_gate<32, 2, 16>(a, s);
  else e = launch_gate<64, 1, 16>(a, s);
  if (e != cudaSuccess) return e;
  Prio pr{};
  if (a.rts) {
    pr.on = 1;
    pr.m = 1;
    while (((int64_t)1 << (2 * pr.m)) < a.T) ++pr.m;
    pr.mask = (1u << pr.m) - 1u;
    const uint32_t lo = (uint32_t)a.seed, hi = (uint32_t)(a.seed >> 32);
    for (int r = 0; r < 4; ++r) pr.k[r] = lo * 0x9E3779B9u + hi + (uint32_t)r * 0x85EBCA6Bu;
  }
  const int nblocks = (int)((a.T * a.K + SCAN_BLOCK - 1) / SCAN_BLOCK);
  slot_local_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.T, a.K, a.E, pr, a.local_rank, a.block_hist);
  slot_final_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.local_rank, a.block_hist, a.T, a.K, a.E,
                                                   a.C, nblocks, pr, a.slot, a.tok_of, a.count, a.load);
  if (a.aux_out) {
    if (a.E <= 8) aux_partial_kernel<8><<<AUX_GRID, 256, 0, s>>>(a.logits, a.expert, a.T, a.K, a.E, a.aux_partial);
    else if (a.E <= 16) aux_partial_kernel<16><<<AUX_GRID, 256, 0, s>>>(a.logits, a.expert, a.T, a.K, a.E, a.aux_partial);
    else if (a.E <= 32) aux_partial_kernel<32><<<AUX_GRID, 256, 0, s>>>(a.logits, a.expert, a.T, a.K, a.E, a.aux_partial);
    else aux_partial_kernel<64><<<AUX_GRID, 256, 0, s>>>(a.logits, a.expert, a.T, a.K, a.E, a.aux_partial);
    aux_final_kernel<<<1, 64, 0, s>>>(a.aux_partial, a.T, a.E, a.aux_coef, a.aux_out);
  }
  return cudaGetLastError();
}

}  // namespace moe
