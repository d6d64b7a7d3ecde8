// route.cu — F1 (top-1 gate) and F2 (capacity slot scan), SURVEY §8(a).
//
// F1 gate: l = x Wg with fp32 accumulation, softmax max/denominator, lowest-index
// argmax, top-2 gap, p = softmax(l)[e*] (R1, R4). The contraction runs on
// the tensor cores (tcgen05, Wg split into three bf16 terms, see gate_tc_kernel), so
// the kernel streams x at HBM speed instead of being bound by CUDA-core FMAs.
//
// F2 slots: slot_t = #{t' < t : e*(t') = e*(t)} (R3), in two passes: (a) per-block
// warp-match ranks + block histogram — for top-1 in token order done by the gate's
// epilogue per 128-token tile, otherwise slot_local_kernel per 1024 items — and
// (b) slot_final_kernel: block prefix per expert, slot/keep decision, count[E], and
// the inverse map tok_of[e][slot] used by the slot-parallel dispatch.
#include <atomic>
#include <cuda.h>
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {


// Routing decision of one token from its E logits (R1, R4, R5; top-2: R22). Returns the
// tie flag (gap < 1e-6) and, for top-1, the chosen expert in *chosen.
template <int EMAX>
__device__ __forceinline__ bool finalize_token(const float (&lv)[EMAX], int64_t tok, int E, int K,
                                               const int32_t* __restrict__ forced,
                                               int32_t* __restrict__ expert, float* __restrict__ prob,
                                               float* __restrict__ gap, int* chosen_out) {
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
    *chosen_out = best;
    return g < 1e-6f;
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
  *chosen_out = chosen;
  return g < 1e-6f;
}

// ---------------------------------------------------------------- F1 on the tensor cores
// l = x . Wg is a [T, H] x [H, E] contraction with E <= 64: tiny N, so the gate is
// bound by streaming x from HBM (2H bytes per token), not by its 2HE flops — as long as
// the flops leave the CUDA cores. x is exact bf16; Wg (fp32) is split into three bf16
// terms hi + mid + lo (24 significant bits, i.e. all of Wg's) by the converter warps, so
// x . Wg = x . hi + x . mid + x . lo with every product exact and fp32 accumulation in
// TMEM: one tcgen05.mma M = 128 rows, N = 3 * NPAD (hi | mid | lo columns), K = 16.
// Precision: a tensor-core accumulation of many MMAs into one fp32 accumulator loses
// bits (measured max logit error 1.2e-5 with one accumulator over K = 2048, 1.4e-6 with
// 10 chunks), so every 64-wide k block gets a fresh accumulator: the MMA issuer writes
// k block i into TMEM chunk buffer i % NB (hi | mid | lo, 3 NPAD columns) and commits it,
// and the epilogue warps — otherwise idle during the main loop — drain each chunk as it
// completes, summing (hi + (mid + lo)) into the token's logits with Kahan compensation,
// then release the buffer. No accumulator holds more than 64 products (error ~1e-7,
// tests/test_gpu_layer.py), so routing matches the oracle outside the 1e-6 tie set.
// A tile holds R <= 128 tokens, R = T / #SMs rounded up to 8, so every SM streams
// (rows >= R of the 128-row MMA are ignored). Measured (tools/read_bw.cu): a cold 64 MiB
// read takes ~18 us with the best LDG.128 kernel and ~20.5 us with 64 x 128 TMA boxes at
// 8 stages, so this kernel's floor is the read of x, not its arithmetic.
//
// Warp roles (320 threads, one CTA per SM, persistent over tiles):
//   warps 0-3  epilogue: TMEM lane quadrant = token row; routing decision per thread
//              (finalize_token), and — top-1 in token order — the F2 block scan of the
//              tile (warp match ranks + tile histogram, H5) so only slot_final remains;
//   warp 4     TMEM allocation, TMA producer: per 64-wide k block the x box (R x 64 bf16,
//              128B swizzle) and the contiguous Wg rows [64][E] fp32 (1-D bulk copy, L2);
//   warp 5     MMA issuer (one elected lane);
//   warps 6-9  Wg converters: fp32 rows -> hi | mid | lo bf16 B tile in the K-major
//              128B-swizzle layout TMA would produce, then fence.proxy.async (no separate
//              split launch; measured: a split kernel + PDL costs ~4 us more per step).
namespace gtc {
constexpr int ROWS = 128;  // UMMA M
constexpr int BKG = 64;    // k per stage (one 128-byte swizzle row of bf16)
constexpr int CONV_WARPS = 4;
constexpr int THREADS = (6 + CONV_WARPS) * 32;
constexpr int TMEM_COLS = 512;

template <int NPAD>
struct Cfg {
  static constexpr int A_BYTES = ROWS * BKG * 2;      // 16 KiB (R rows used)
  static constexpr int B_BYTES = 3 * NPAD * BKG * 2;  // hi | mid | lo rows, 128 B each
  static constexpr int W_BYTES = BKG * NPAD * 4;      // fp32 Wg rows [64][E], E <= NPAD
  static constexpr int STAGE = A_BYTES + B_BYTES + W_BYTES;
  static constexpr int STAGES = (200 * 1024 / STAGE) < 8 ? (200 * 1024 / STAGE) : 8;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int NCOL = 3 * NPAD;  // hi | mid | lo columns of one chunk
  static constexpr int NB = TMEM_COLS / NCOL;  // chunk buffers in TMEM (one k block each)
  static_assert(STAGE % 1024 == 0 && STAGES >= 3 && NCOL % 16 == 0 && NCOL <= 256, "gate tile");
};

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

struct Args {
  const float* wg;
  const int32_t* forced;
  int64_t T;
  int H, E, K, R;
  int fuse_scan;  // top-1, token order: the epilogue produces local_rank / tile histogram
  float* logits;
  int32_t* expert;
  float* prob;
  float* gap;
  int32_t* local_rank;  // [T]
  int32_t* tile_hist;   // [ntiles][E]
  int32_t* tile_ties;   // [ntiles]
};

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, float (&r)[16]) {
  uint32_t u[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
      : "r"(taddr));
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = __uint_as_float(u[i]);
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

template <int NPAD>
__global__ void __launch_bounds__(THREADS, 1)
    gate_tc_kernel(const __grid_constant__ CUtensorMap tmX, const Args a) {
  using C = Cfg<NPAD>;
  constexpr int S = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int NB = C::NB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::STAGE);
  // [0,S) full (x landed), [S,2S) bready (B tile converted), [2S,3S) empty (MMAs done
  // with the stage), [3S,3S+NB) chunk full, [3S+NB,3S+2NB) chunk empty (drained)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 2 * NB);
  __shared__ int32_t wh[4][64];  // fused scan: per-warp expert histogram
  __shared__ int32_t wties[4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = a.H / BKG;
  const int R = a.R;
  const int64_t ntiles = (a.T + R - 1) / R;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[S + s]), CONV_WARPS);
      mbar_init(smem_u32(&bars[2 * S + s]), 1);
    }
    for (int c = 0; c < NB; ++c) {
      mbar_init(smem_u32(&bars[3 * S + c]), 1);
      mbar_init(smem_u32(&bars[3 * S + NB + c]), 4);
    }
    fence_barrier_init();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the slot scan may be scheduled now; it waits for this grid's completion itself
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 4) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbytes = (uint32_t)(BKG * a.E * 4);
      const uint32_t bytes = (uint32_t)(R * BKG * 2) + wbytes;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(smem_u32(&bars[2 * S + stage]), phase ^ 1);
          const uint32_t full = smem_u32(&bars[stage]);
          const uint32_t st = smem_u32(smem + stage * C::STAGE);
          mbar_arrive_expect_tx(full, bytes);
          tma_load_3d(st, &tmX, full, kb * BKG, (int)(tile * R), 0);
          bulk_load(st + C::A_BYTES + C::B_BYTES, a.wg + (size_t)kb * BKG * a.E, wbytes, full);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(C::NCOL >> 3) << 17) |
                                 ((uint32_t)(ROWS >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;  // k blocks issued by this CTA (chunk buffer g % NB, use g / NB)
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int buf = g % NB;
          mbar_wait(smem_u32(&bars[3 * S + NB + buf]), ((g / NB) & 1) ^ 1);  // drained
          mbar_wait(smem_u32(&bars[stage]), phase);
          mbar_wait(smem_u32(&bars[S + stage]), phase);
          tc_fence_after();
          const uint32_t ab = smem_u32(smem + stage * C::STAGE);
          const uint32_t bb = ab + C::A_BYTES;
#pragma unroll
          for (int j = 0; j < BKG / 16; ++j)
            tc_mma_f16(tmem_base + buf * C::NCOL, sw128_desc(ab + j * 32), sw128_desc(bb + j * 32), idesc,
                       j == 0 ? 0u : 1u);
          tc_commit(smem_u32(&bars[2 * S + stage]));
          tc_commit(smem_u32(&bars[3 * S + buf]));
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 6) {
    // ---------------------------------------------------------- Wg converters
    // (n, j): expert row n, 16-byte chunk j (k = 8 j .. 8 j + 7) of the 128-byte row
    const int ct = threadIdx.x - 6 * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(smem_u32(&bars[stage]), phase);  // Wg rows (and x) of this stage landed
        uint8_t* st = smem + stage * C::STAGE;
        const float* w = reinterpret_cast<const float*>(st + C::A_BYTES + C::B_BYTES);
        const uint32_t bb = smem_u32(st + C::A_BYTES);
        for (int q = ct; q < NPAD * 8; q += CONV_WARPS * 32) {
          const int n = q % NPAD, j = q / NPAD;
          uint32_t hw[4], mw[4], lw[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            bf16 h[2], m[2], l[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float v = n < a.E ? w[(8 * j + 2 * p + u) * a.E + n] : 0.f;
              h[u] = __float2bfloat16_rn(v);
              const float r1 = v - __bfloat162float(h[u]);
              m[u] = __float2bfloat16_rn(r1);
              l[u] = __float2bfloat16_rn(r1 - __bfloat162float(m[u]));
            }
            hw[p] = pack2(h[0], h[1]);
            mw[p] = pack2(m[0], m[1]);
            lw[p] = pack2(l[0], l[1]);
          }
          const uint32_t off = (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4));
          st_shared_v4(bb + off, hw[0], hw[1], hw[2], hw[3]);
          st_shared_v4(bb + NPAD * 128 + off, mw[0], mw[1], mw[2], mw[3]);
          st_shared_v4(bb + 2 * NPAD * 128 + off, lw[0], lw[1], lw[2], lw[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars[S + stage]));
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue (warps 0-3)
    int g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      float lv[NPAD], comp[NPAD];  // Kahan sum over the k-block chunks
#pragma unroll
      for (int e = 0; e < NPAD; ++e) { lv[e] = 0.f; comp[e] = 0.f; }
      const uint32_t trow = tmem_base + ((uint32_t)(warp * 32) << 16);
      for (int kb = 0; kb < KB; ++kb, ++g) {
        const int buf = g % NB;
        mbar_wait(smem_u32(&bars[3 * S + buf]), (g / NB) & 1);
        tc_fence_after();
        if (warp * 32 < R) {  // warp-uniform: quadrants past the tile's rows hold nothing
#pragma unroll
          for (int nb = 0; nb < NPAD / 16; ++nb) {
            float h[16], m[16], l[16];
            const uint32_t c0 = trow + buf * C::NCOL + nb * 16;
            tmem_ld_x16(c0, h);
            tmem_ld_x16(c0 + NPAD, m);
            tmem_ld_x16(c0 + 2 * NPAD, l);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int e = nb * 16 + i;
              const float y = (h[i] + (m[i] + l[i])) - comp[e];
              const float t = lv[e] + y;
              comp[e] = (t - lv[e]) - y;
              lv[e] = t;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars[3 * S + NB + buf]));  // chunk drained
      }

      const int row = warp * 32 + lane;
      const int64_t tok = tile * R + row;
      const bool valid = row < R && tok < a.T;
      bool tie = false;
      int chosen = -1;
      if (valid) {
        float* lrow = a.logits + (size_t)tok * a.E;
        if ((a.E & 3) == 0) {
#pragma unroll
          for (int e = 0; e < NPAD; e += 4)
            if (e < a.E) *reinterpret_cast<float4*>(lrow + e) = make_float4(lv[e], lv[e + 1], lv[e + 2], lv[e + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < NPAD; ++e)
            if (e < a.E) lrow[e] = lv[e];
        }
        tie = finalize_token<NPAD>(lv, tok, a.E, a.K, a.forced, a.expert, a.prob, a.gap, &chosen);
      }
      const int nt = __popc(__ballot_sync(0xffffffffu, tie));
      if (lane == 0) wties[warp] = nt;
      int rk = 0;  // rank among this warp's tokens routed to the same expert
      if (a.fuse_scan) {
        for (int e = lane; e < 64; e += 32) wh[warp][e] = 0;
        __syncwarp();
        const int e = valid ? chosen : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, e);
        rk = __popc(peers & ((1u << lane) - 1));
        if (e >= 0 && rk == 0) wh[warp][e] = __popc(peers);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (a.fuse_scan) {
        if (valid) {
          int base = 0;
          for (int w = 0; w < warp; ++w) base += wh[w][chosen];
          a.local_rank[tok] = base + rk;
        }
        const int t = threadIdx.x;
        if (t < a.E) a.tile_hist[(size_t)tile * a.E + t] = wh[0][t] + wh[1][t] + wh[2][t] + wh[3][t];
      }
      if (threadIdx.x == 0) a.tile_ties[tile] = wties[0] + wties[1] + wties[2] + wties[3];
      asm volatile("bar.sync 1, 128;" ::: "memory");  // wh / wties reused by the next tile
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}
}  // namespace gtc

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
// CTA 0 also sums the gate tiles' tie counts into *ties.
__global__ void __launch_bounds__(SCAN_BLOCK)
    slot_final_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ local_rank,
                      const int32_t* __restrict__ block_hist, int64_t T, int K, int E, int64_t C,
                      int nblocks, Prio pr, const int32_t* __restrict__ tile_ties, int ntiles,
                      int32_t* __restrict__ ties, int32_t* __restrict__ slot, int32_t* __restrict__ tok_of,
                      int32_t* __restrict__ count, int32_t* __restrict__ load) {
  __shared__ int32_t prefix[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < E; e += SCAN_BLOCK / 32) {  // one warp per expert
    int run = 0, total = 0;
    for (int b = lane; b < nblocks; b += 32) {
      const int c = block_hist[(size_t)b * E + e];
      if (b < (int)blockIdx.x) run += c;
      total += c;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      run += __shfl_xor_sync(0xffffffffu, run, o);
      total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if (lane == 0) {
      prefix[e] = run;
      if (blockIdx.x == 0) {
        load[e] = total;
        count[e] = (int)((int64_t)total < C ? total : C);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x >= 32 * 31) {  // last warp: tie total, fixed order
    int n = 0;
    for (int b = threadIdx.x & 31; b < ntiles; b += 32) n += tile_ties[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0) *ties = n;
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

// (b') fused mode: one CTA per gate tile of R tokens (token order, top-1); the tile
// histograms come from the gate's epilogue.
__global__ void __launch_bounds__(1024)
    slot_final_tiles_kernel(const int32_t* __restrict__ expert, const int32_t* __restrict__ local_rank,
                            const int32_t* __restrict__ tile_hist, int64_t T, int E, int64_t C, int R, int ntiles,
                            const int32_t* __restrict__ tile_ties, int32_t* __restrict__ ties,
                            int32_t* __restrict__ slot, int32_t* __restrict__ tok_of, int32_t* __restrict__ count,
                            int32_t* __restrict__ load) {
  __shared__ int32_t prefix[64];
  // launched as a programmatic dependent of the gate: everything above overlaps its tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tile = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = warp; e < E; e += nwarps) {  // one warp per expert
    int run = 0, total = 0;
    for (int b = lane; b < ntiles; b += 32) {
      const int c = tile_hist[(size_t)b * E + e];
      if (b < tile) run += c;
      total += c;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      run += __shfl_xor_sync(0xffffffffu, run, o);
      total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if (lane == 0) {
      prefix[e] = run;
      if (tile == 0) {
        load[e] = total;
        count[e] = (int)((int64_t)total < C ? total : C);
      }
    }
  }
  if (tile == 0 && warp == 0) {  // tie total, fixed order
    int n = 0;
    for (int b = lane; b < ntiles; b += 32) n += tile_ties[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) *ties = n;
  }
  __syncthreads();
  const int64_t t = (int64_t)tile * R + threadIdx.x;
  if ((int)threadIdx.x >= R || t >= T) return;
  const int e = expert[t];
  const int64_t sl = (int64_t)prefix[e] + local_rank[t];
  if (sl < C) {
    slot[t] = (int32_t)sl;
    tok_of[(size_t)e * C + sl] = (int32_t)t;
  } else {
    slot[t] = -1;
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

template <int NPAD>
cudaError_t launch_gate_tc(const RouteArgs& a, bool fuse, int* R_out, cudaStream_t s) {
  using Cf = gtc::Cfg<NPAD>;
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(gtc::gate_tc_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int sms = 0;
  CUtensorMap tm;
  e = tensor_map_bf16(&tm, a.x, (uint64_t)a.H, (uint64_t)a.T, gtc::BKG, 8, &sms);  // sms (box re-encoded below)
  if (e != cudaSuccess) return e;
  // R tokens per tile: every SM gets a tile (R a multiple of 8, at most the MMA's 128 rows)
  int64_t R = (a.T + sms - 1) / sms;
  R = (R + 7) & ~7;
  if (R > gtc::ROWS) R = gtc::ROWS;
  e = tensor_map_bf16(&tm, a.x, (uint64_t)a.H, (uint64_t)a.T, gtc::BKG, (uint32_t)R, &sms);
  if (e != cudaSuccess) return e;
  gtc::Args g;
  g.wg = a.wg; g.forced = a.forced; g.T = a.T; g.H = a.H; g.E = a.E; g.K = a.K; g.R = (int)R;
  g.fuse_scan = fuse ? 1 : 0;
  g.logits = a.logits; g.expert = a.expert; g.prob = a.prob; g.gap = a.gap;
  g.local_rank = a.local_rank; g.tile_hist = a.block_hist; g.tile_ties = a.tile_ties;
  const int64_t ntiles = (a.T + R - 1) / R;
  *R_out = (int)R;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ntiles < sms ? ntiles : sms));
  cfg.blockDim = dim3(gtc::THREADS);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = s;
  return cudaLaunchKernelEx(&cfg, gtc::gate_tc_kernel<NPAD>, tm, g);
}

}  // namespace

cudaError_t route(const RouteArgs& a, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (a.T == 0) {
    e = cudaMemsetAsync(a.ties, 0, sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.E, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.load, 0, sizeof(int32_t) * a.E, s);
    if (e == cudaSuccess && a.aux_out) e = cudaMemsetAsync(a.aux_out, 0, sizeof(float) * (a.E + 1), s);
    return e;
  }
  // top-1 in token order: the gate's epilogue does the block half of the slot scan
  const bool fuse = a.K == 1 && !a.rts;
  int R = 0;
  if (a.E <= 16) e = launch_gate_tc<16>(a, fuse, &R, s);
  else if (a.E <= 32) e = launch_gate_tc<32>(a, fuse, &R, s);
  else e = launch_gate_tc<64>(a, fuse, &R, s);
  if (e != cudaSuccess) return e;
  const int ntiles = (int)((a.T + R - 1) / R);
  if (fuse) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ntiles);
    cfg.blockDim = dim3(32 * (a.E < 4 ? 4 : a.E > 32 ? 32 : a.E));
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, slot_final_tiles_kernel, (const int32_t*)a.expert, (const int32_t*)a.local_rank,
                           (const int32_t*)a.block_hist, a.T, a.E, a.C, R, ntiles, (const int32_t*)a.tile_ties,
                           a.ties, a.slot, a.tok_of, a.count, a.load);
    if (e != cudaSuccess) return e;
  } else {
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
    slot_final_kernel<<<nblocks, SCAN_BLOCK, 0, s>>>(a.expert, a.local_rank, a.block_hist, a.T, a.K, a.E, a.C,
                                                     nblocks, pr, a.tile_ties, ntiles, a.ties, a.slot, a.tok_of,
                                                     a.count, a.load);
  }
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
