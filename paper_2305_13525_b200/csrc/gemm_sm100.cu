// gemm_sm100.cu — the expert FFN contraction on 5th-gen tensor cores.
//
// Batched bf16 GEMM D[b] = epi(A[b] . B[b]^T), fp32 accumulation in TMEM.
// Every expert GEMM of the layer is one launch:
// capacity padding gives every local expert the same R = G_expert*C rows
// (SURVEY §7 H2), so the "grouped" GEMM is a uniform batch with the expert as
// the third TMA coordinate.
//
// Design (sm_100a):
//  * persistent, a CTA pair (cluster of 2) per 2 SMs, 256x256 output tile with
//    tcgen05.mma.cta_group::2 (M = 256), BK = 64, 6-stage TMA -> smem ring (128B
//    swizzle), mbarrier full/empty pipeline;
//  * warp 0: TMA producer (one elected lane); warp 1: tcgen05.mma issuer (leader
//    CTA, one lane); warp 2: TMEM allocator; warps 4+: epilogue (tcgen05.ld ->
//    fp32 epilogue -> bf16 -> global);
//  * TMEM holds two 128x256 fp32 accumulators per CTA (512 columns) so the
//    epilogue of tile i overlaps the main loop of tile i+1;
//  * operands may be K-major or MN-major (instruction-descriptor bits), which
//    covers the forward (X W1^T, A W2^T), the data-gradient (dY W2, dH W1)
//    and the weight-gradient (dY^T A, dH^T X) GEMMs without transposes;
//  * epilogues: plain store; GeLU (stores G = gelu'(Hpre) for the backward and
//    A = gelu(Hpre)); dGeLU (multiplies by G read from global) — the backward's
//    dGeLU becomes one multiply and Hpre itself is never stored.
//  * no split-K: a row's result never depends on its position, which DTD's
//    bitwise-equality property relies on.
#include <atomic>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int BM = 128;  // rows of A per CTA (the CTA pair covers 256)
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int TMEM_COLS = 512;        // 2 accumulators x 256 fp32 columns

struct Params {
  int batch, M, N, K;
  int tiles_m, tiles_n, total_tiles, k_blocks;
  int64_t d_bs;  // elements between batches of D / aux
  int k_main;    // EPI_SCATTER: k-blocks of the main operands (the last one is the extension)
  bf16* D;
  bf16* aux;
  GateDxArgs g;  // EPI_SCATTER / EPI_COMBINE
  GemmSignal sig;  // sig.cnt != null: per-part completion flags (EPI_STORE)
  PeerOut po;      // po.table != null: rows into the source ranks' windows (EPI_STORE)
};

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// ---------------------------------------------------------------- 2-CTA variant
// A CTA pair (cluster of 2) computes a 256 x 256 tile with tcgen05.mma.cta_group::2
// (M = 256): each CTA stages its 128 rows of A and its 128 rows of B per
// k-block (32 KiB / stage, 6 stages), so per-SM shared-memory traffic per MMA
// is halved versus the 1-CTA 128 x 256 tile. The leader (rank 0) issues the
// MMAs; both CTAs' TMA loads count on the leader's full barrier; commits are
// multicast to both CTAs; each CTA's epilogue drains its own 128 TMEM lanes and
// both arrive on the leader's tmem-empty barrier.
constexpr int A2_STAGE = 128 * BK * 2;  // 16 KiB
constexpr int B2_STAGE = 128 * BK * 2;  // 16 KiB (this CTA's half of BN = 256)
constexpr int STAGES2 = 6;
constexpr int EPI_BUF = 32 * 32 * 2;  // one warp's 32 x 32 bf16 chunk, 64B-swizzled
// Epilogue warps: 4 per 64 columns (one per TMEM lane quadrant). The plain
// epilogue uses 16 (each warp drains 32 rows x 64 columns per tile); the GeLU
// (two outputs, ~160 registers) and dGeLU (a lane-per-row read of G per chunk)
// epilogues use 8 (32 rows x 128 columns) — measured: dGeLU 0.577 -> 0.552 Mcycles.
__host__ __device__ constexpr int epi_outs(int epi) { return (epi == EPI_GELU || epi == EPI_COMBINE) ? 2 : 1; }
__host__ __device__ constexpr int epi_warps(int epi) { return (epi == EPI_STORE || epi == EPI_SCATTER) ? 16 : 8; }
constexpr int GDX_EMAX = 16;  // EPI_SCATTER: experts covered by the 64-wide K extension (3 x 16 + pad)
__host__ __device__ constexpr int threads2(int epi) { return (4 + epi_warps(epi)) * 32; }
__host__ __device__ constexpr int epi_smem(int epi) { return epi_warps(epi) * epi_outs(epi) * EPI_BUF; }
__host__ __device__ constexpr int smem2_bytes(int epi) {
  return STAGES2 * (A2_STAGE + B2_STAGE) + epi_smem(epi) + 1024 + 256;
}
static_assert(smem2_bytes(EPI_STORE) <= 227 * 1024 && smem2_bytes(EPI_GELU) <= 227 * 1024 &&
              smem2_bytes(EPI_COMBINE) <= 227 * 1024, "smem");

__host__ __device__ constexpr uint32_t instr_desc_m256(int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// Development instrumentation (tools/gemm_prof.cu builds this file with MOE_GEMM_PROF):
// per-CTA cycle counters of the pipeline waits. Compiled out of the library.
#ifdef MOE_GEMM_PROF
__device__ unsigned long long g_prof[160][8];
#define PROF_T0(v) const long long v = clock64()
#define PROF_ADD(i, t0) atomicAdd(&g_prof[blockIdx.x][i], (unsigned long long)(clock64() - (t0)))
#define PROF_CNT(i) atomicAdd(&g_prof[blockIdx.x][i], 1ull)
#else
#define PROF_CNT(i)
#define PROF_T0(v)
#define PROF_ADD(i, t0)
#endif

template <int A_MN, int B_MN, int EPI>
__global__ void __launch_bounds__(threads2(EPI), 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                 const Params p) {
  constexpr int EW = epi_warps(EPI);
  constexpr int NO = epi_outs(EPI);
  constexpr int COLS_W = BN / (EW / 4);  // columns one epilogue warp drains per tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES2 * A2_STAGE;
  uint8_t* smE = smB + STAGES2 * B2_STAGE;  // epilogue transpose buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(smE + epi_smem(EPI));
  // [0,S) full (leader's counts both CTAs), [S,2S) empty, [2S,2S+2) tmem_full, [2S+2,2S+4) tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES2 + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  PROF_T0(t_start);
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[STAGES2 + s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&bars[2 * STAGES2 + a]), 1);
      mbar_init(smem_u32(&bars[2 * STAGES2 + 2 + a]), 2 * EW);  // epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int tiles_mn = p.tiles_m * p.tiles_n;
  // Programmatic dependent launch: the prologue above (barriers, TMEM, descriptor
  // prefetch) may overlap the tail of the previous kernel in the stream; every global
  // access below waits for its completion, and the next kernel may be scheduled as
  // this grid's CTAs exit.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < p.total_tiles; tile += nclusters) {
        const int b = tile / tiles_mn;
        const int r = tile - b * tiles_mn;
        const int m0 = (r / p.tiles_n) * 256 + rank * 128;
        const int n0 = (r % p.tiles_n) * BN + rank * 128;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          PROF_T0(w0);
          mbar_wait(smem_u32(&bars[STAGES2 + stage]), phase ^ 1);
          PROF_ADD(0, w0);
          const uint32_t full = smem_u32(&bars[stage]);
          if (leader) mbar_arrive_expect_tx(full, 2 * (A2_STAGE + B2_STAGE));
          const uint32_t a_dst = smem_u32(smA + stage * A2_STAGE);
          const uint32_t b_dst = smem_u32(smB + stage * B2_STAGE);
          const int k0 = kb * BK;
          if (EPI == EPI_SCATTER && kb >= p.k_main) {
            // K extension (B10's gate term): A2 = [E][M][64] bf16 K-major, B2 = [64][N]
            // bf16 MN-major, shared by every batch
            tma_load_3d_2sm(a_dst, &tmA2, full, 0, m0, b);
            tma_load_3d_2sm(b_dst, &tmB2, full, n0, 0, 0);
            tma_load_3d_2sm(b_dst + 8192, &tmB2, full, n0 + 64, 0, 0);
          } else {
            if (A_MN) {
              tma_load_3d_2sm(a_dst, &tmA, full, m0, k0, b);
              tma_load_3d_2sm(a_dst + 8192, &tmA, full, m0 + 64, k0, b);
            } else {
              tma_load_3d_2sm(a_dst, &tmA, full, k0, m0, b);
            }
            if (B_MN) {
              tma_load_3d_2sm(b_dst, &tmB, full, n0, k0, b);
              tma_load_3d_2sm(b_dst + 8192, &tmB, full, n0 + 64, k0, b);
            } else {
              tma_load_3d_2sm(b_dst, &tmB, full, k0, n0, b);
            }
          }
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = instr_desc_m256(A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int tile = cluster; tile < p.total_tiles; tile += nclusters, ++iter) {
        const int acc = iter & 1;
        const uint32_t acc_phase = (iter >> 1) & 1;
        PROF_T0(w2);
        mbar_wait(smem_u32(&bars[2 * STAGES2 + 2 + acc]), acc_phase ^ 1);
        PROF_ADD(2, w2);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          PROF_T0(w1);
          mbar_wait(smem_u32(&bars[stage]), phase);
          PROF_ADD(1, w1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * A2_STAGE);
          const uint32_t b_base = smem_u32(smB + stage * B2_STAGE);
#pragma unroll
          for (int j = 0; j < BK / 16; ++j) {
            const uint64_t ad = A_MN ? smem_desc(a_base + j * 2048, 8192, 1024)
                                     : smem_desc(a_base + j * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(b_base + j * 2048, 8192, 1024)
                                     : smem_desc(b_base + j * 32, 16, 1024);
            tc_mma_f16_2sm(tmem_d, ad, bd, idesc, (kb | j) != 0);
          }
          tc_commit_2sm(smem_u32(&bars[STAGES2 + stage]), 0x3);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm(smem_u32(&bars[2 * STAGES2 + acc]), 0x3);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // TMEM -> registers (lane = row, 32 fp32 columns) -> epilogue math -> bf16 ->
    // this warp's 64B-swizzled 32 x 32 smem buffer -> read back 8 rows x 64 B per
    // instruction -> st.global.v4 (full 32 B sectors). Rows >= M and columns >= N
    // are skipped. No async proxy on the store side: a chunk costs two __syncwarp.
    const int ew = warp - 4;
    const int quad = warp & 3;              // TMEM lane quadrant this warp may access
    const int col0 = (ew >> 2) * COLS_W;    // this warp's column slice of the tile
    const uint32_t bD = smem_u32(smE) + ew * NO * EPI_BUF;
    const uint32_t bX = bD + EPI_BUF;
    const uint32_t swz = (uint32_t)((lane >> 1) & 3);
    const int rr = lane >> 2, qq = lane & 3;  // read-back: row within an 8-row group, 16 B piece
    int iter = 0;
    for (int tile = cluster; tile < p.total_tiles; tile += nclusters, ++iter) {
      const int b = tile / tiles_mn;
      const int r = tile - b * tiles_mn;
      const int m0 = (r / p.tiles_n) * 256 + rank * 128;
      const int n0 = (r % p.tiles_n) * BN;
      const int acc = iter & 1;
      const uint32_t acc_phase = (iter >> 1) & 1;
      PROF_T0(w3);
      mbar_wait(smem_u32(&bars[2 * STAGES2 + acc]), acc_phase);
      if (ew == 0 && lane == 0) PROF_ADD(3, w3);
      PROF_T0(w4);
      tc_fence_after();
      const int mrow0 = m0 + quad * 32;
      const int m = mrow0 + lane;
      const bool row_ok = m < p.M;
      const size_t row_off = (size_t)b * p.d_bs + (size_t)(row_ok ? m : 0) * (size_t)p.N;
      int tok = -1;                 // EPI_SCATTER / EPI_COMBINE: token of this lane's slot row (-1: empty)

      float pscale = 0.f;           // EPI_COMBINE: p_t of that token
      if (EPI == EPI_COMBINE) {
        tok = (row_ok && m < p.g.count[b]) ? p.g.tok_of[(size_t)b * p.g.C + m] : -1;
        pscale = tok >= 0 ? p.g.prob[tok] : 0.f;
      }
      if (EPI == EPI_SCATTER) tok = (row_ok && m < p.g.count[b]) ? p.g.tok_of[(size_t)b * p.g.C + m] : -1;
#pragma unroll 1
      for (int c = col0; c < col0 + COLS_W; c += 32) {
        const int n = n0 + c;
        if (n >= p.N) break;  // uniform across the warp
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + c, v);
        uint4 hpre[4];
        if (EPI == EPI_DGELU) {
          const bf16* hsrc = p.aux + row_off + n;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            hpre[q] = row_ok ? *reinterpret_cast<const uint4*>(hsrc + q * 8) : make_uint4(0, 0, 0, 0);
        }
        tmem_wait_ld();
        uint32_t o[16], g[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) {
          const float2 f = make_float2(__uint_as_float(v[2 * w]), __uint_as_float(v[2 * w + 1]));
          if (EPI == EPI_DGELU) {
            // aux holds gelu'(Hpre) (stored by the forward GeLU epilogue)
            const uint32_t hw = (w & 3) == 0 ? hpre[w >> 2].x : (w & 3) == 1 ? hpre[w >> 2].y
                              : (w & 3) == 2 ? hpre[w >> 2].z : hpre[w >> 2].w;
            const float2 r2 = f2mul(f, unpack_bf16x2(hw));
            o[w] = pack_bf16x2(r2.x, r2.y);
          } else if (EPI == EPI_GELU) {
            // D = gelu'(acc) (for the backward), aux = gelu(acc) (the FFN activation)
            float2 gg, gp;
            gelu_and_grad2(f, gg, gp);
            o[w] = pack_bf16x2(gp.x, gp.y);
            g[w] = pack_bf16x2(gg.x, gg.y);
          } else if (EPI == EPI_COMBINE) {
            o[w] = pack_bf16x2(f.x, f.y);                    // O (slot space, for the backward)
            g[w] = pack_bf16x2(pscale * f.x, pscale * f.y);  // y row of the token
          } else {
            o[w] = pack_bf16x2(f.x, f.y);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t off = lane * 64 + ((q ^ swz) << 4);
          st_shared_v4(bD + off, o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
          if (EPI == EPI_GELU || EPI == EPI_COMBINE)
            st_shared_v4(bX + off, g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
        }
        __syncwarp();
        const bool col_ok = n + qq * 8 < p.N;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 8 + rr;
          const uint32_t off = row * 64 + ((qq ^ ((row >> 1) & 3)) << 4);
          const int mm = mrow0 + row;
          const bool ok = mm < p.M && col_ok;
          const size_t go = (size_t)b * p.d_bs + (size_t)mm * (size_t)p.N + n + qq * 8;
          const uint4 vd = ld_shared_v4(bD + off);
          if (EPI == EPI_SCATTER) {  // scatter to the token's dx row
            const int trow = __shfl_sync(0xffffffffu, tok, row);
            if (trow >= 0 && col_ok)
              st_v4(static_cast<bf16*>(p.g.dx) + (size_t)trow * p.N + n + qq * 8, vd);
          } else if (ok) {
            if (EPI == EPI_STORE && p.po.table) {  // F9 fused: the row goes to its source rank
              const int64_t sblk = mm / p.po.C;
              bf16* base = static_cast<bf16*>(p.po.table[(p.po.rank0 + sblk) * p.po.nwin + p.po.win]);
              st_v4(base + ((size_t)(p.po.e0 + b) * p.po.C + (mm - sblk * p.po.C)) * p.N + n + qq * 8, vd);
            } else {
              st_v4(p.D + go, vd);
            }
          }
          if (EPI == EPI_GELU) {
            const uint4 vx = ld_shared_v4(bX + off);
            if (ok) st_v4(p.aux + go, vx);
          }
          if (EPI == EPI_COMBINE) {  // scatter the weighted row to y
            const uint4 vx = ld_shared_v4(bX + off);
            const int trow = __shfl_sync(0xffffffffu, tok, row);
            if (trow >= 0 && col_ok) st_v4(static_cast<bf16*>(p.g.dx) + (size_t)trow * p.N + n + qq * 8, vx);
          }
        }
        __syncwarp();  // the buffer is rewritten by the next chunk
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(smem_u32(&bars[2 * STAGES2 + 2 + acc]), 0);
      if (EPI == EPI_STORE && p.sig.cnt) {
        // every epilogue warp of this CTA has stored its rows of the tile
        asm volatile("bar.sync 1, %0;" ::"r"(EW * 32) : "memory");
        if (ew == 0 && lane == 0) {
          int q = 0;
          while (q + 1 < p.sig.nparts && b >= p.sig.part_b[q + 1]) ++q;
          const int target = (p.sig.part_b[q + 1] - p.sig.part_b[q]) * tiles_mn * 2;
          __threadfence_system();
          if (atomicAdd(&p.sig.cnt[q], 1) == target - 1) {
            p.sig.cnt[q] = 0;
            __threadfence_system();
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.sig.flag + q), "r"(p.sig.epoch) : "memory");
          }
        }
      }
      if (ew == 0 && lane == 0) { PROF_ADD(4, w4); PROF_CNT(6); }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (threadIdx.x == 0) PROF_ADD(5, t_start);
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
const bool g_pdl = [] {  // MOE_NO_PDL=1: plain stream serialization (A/B)
  const char* e = std::getenv("MOE_NO_PDL");
  return !(e && e[0] == '1');
}();
int g_num_sms = 0;
std::once_flag g_once;
cudaError_t g_init_err = cudaSuccess;

void init_once() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  g_init_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (g_init_err == cudaSuccess && q != cudaDriverEntryPointSuccess) g_init_err = cudaErrorNotSupported;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int dev = 0;
  if (g_init_err == cudaSuccess) g_init_err = cudaGetDevice(&dev);
  if (g_init_err == cudaSuccess)
    g_init_err = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
}

// 3-D bf16 tensor map {inner, outer, batch}, box {box_inner, box_outer, 1}.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t batch,
              uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B, uint64_t batch_stride = 0) {
  cuuint64_t dims[3] = {inner, outer, batch};
  cuuint64_t strides[2] = {inner * 2, (batch_stride ? batch_stride : inner * outer) * 2};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int A_MN, int B_MN, int EPI>
cudaError_t launch2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ta2, const CUtensorMap& tb2,
                    const Params& p, cudaStream_t s) {
  static std::atomic<bool> attr{false};  // idempotent; ranks may launch from several threads
  auto k = gemm2_kernel<A_MN, B_MN, EPI>;
  constexpr int SMEM2_BYTES = smem2_bytes(EPI);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int clusters = g_num_sms / 2;
  if (p.total_tiles < clusters) clusters = p.total_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(threads2(EPI));
  cfg.dynamicSmemBytes = SMEM2_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, ta, tb, ta2, tb2, p);
}

}  // namespace

cudaError_t tensor_map_bf16(void* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                            uint32_t box_outer, int* sms) {
  std::call_once(g_once, init_once);
  if (g_init_err != cudaSuccess) return g_init_err;
  *sms = g_num_sms;
  return make_map(static_cast<CUtensorMap*>(map), ptr, inner, outer, 1, box_inner, box_outer)
             ? cudaSuccess
             : cudaErrorInvalidValue;
}

cudaError_t gemm_tc(const GemmArgs& a, cudaStream_t s, const char** why) {
  std::call_once(g_once, init_once);
  if (g_init_err != cudaSuccess) { *why = "driver entry point / device query failed"; return g_init_err; }
  if (a.batch <= 0 || a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaSuccess;
  if ((a.a_bs || a.d_bs) && a.a_mn) {
    *why = "batch strides need a K-major A";
    return cudaErrorNotSupported;
  }
  CUtensorMap ta, tb;
  bool ok = a.a_mn ? make_map(&ta, a.A, a.M, a.K, a.batch, 64, 64)
                   : make_map(&ta, a.A, a.K, a.M, a.batch, 64, BM, CU_TENSOR_MAP_SWIZZLE_128B,
                              (uint64_t)a.a_bs);
  ok = ok && (a.b_mn ? make_map(&tb, a.B, a.N, a.K, a.batch, 64, 64)
                     : make_map(&tb, a.B, a.K, a.N, a.batch, 64, 128));
  if (!ok) { *why = "cuTensorMapEncodeTiled rejected the operand layout"; return cudaErrorInvalidValue; }
  Params p;
  p.batch = a.batch; p.M = a.M; p.N = a.N; p.K = a.K;
  p.d_bs = a.d_bs ? a.d_bs : (int64_t)a.M * a.N;
  p.tiles_m = (a.M + 255) / 256;
  p.tiles_n = (a.N + BN - 1) / BN;
  p.total_tiles = p.tiles_m * p.tiles_n * a.batch;
  p.k_blocks = (a.K + BK - 1) / BK;
  p.D = static_cast<bf16*>(a.D);
  p.aux = static_cast<bf16*>(a.aux);
  p.g = a.gdx ? *a.gdx : GateDxArgs{};
  p.po = PeerOut{};
  if (a.po) {
    if (a.epilogue != EPI_STORE || a.a_bs || a.d_bs || a.po->C <= 0) {
      *why = "fused return: plain epilogue, dense batches";
      return cudaErrorNotSupported;
    }
    p.po = *a.po;
  }
  p.sig = GemmSignal{};
  if (a.sig) {
    if (a.epilogue != EPI_STORE || a.sig->nparts < 1 || a.sig->nparts > 4 || a.sig->part_b[a.sig->nparts] != a.batch) {
      *why = "completion signal: plain epilogue, 1-4 parts covering the batch";
      return cudaErrorNotSupported;
    }
    p.sig = *a.sig;
  }
  if (a.epilogue == EPI_COMBINE && !a.gdx) {
    *why = "combine epilogue needs its gate arguments";
    return cudaErrorNotSupported;
  }
  CUtensorMap ta2 = ta, tb2 = tb;
  p.k_main = p.k_blocks;
  if (a.epilogue == EPI_SCATTER) {
    if (!a.gdx || !a.b_mn || a.a_mn || !a.gdx->a_ext || !a.gdx->b_ext || a.a_bs || a.d_bs) {
      *why = "scatter epilogue: K-major A, MN-major B, extension operands";
      return cudaErrorNotSupported;
    }
    // A2 = [batch][M][64], B2 = [64][N] (one copy, batch coordinate 0)
    bool ok2 = make_map(&ta2, a.gdx->a_ext, 64, a.M, a.batch, 64, BM) &&
               make_map(&tb2, a.gdx->b_ext, a.N, 64, 1, 64, 64);
    if (!ok2) { *why = "cuTensorMapEncodeTiled rejected the extension operands"; return cudaErrorInvalidValue; }
    p.k_blocks += 1;
  }
  const int key = a.a_mn * 100 + a.b_mn * 10 + a.epilogue;
  switch (key) {
    case 0:   return launch2<0, 0, EPI_STORE>(ta, tb, ta, tb, p, s);
    case 1:   return launch2<0, 0, EPI_GELU>(ta, tb, ta, tb, p, s);
    case 4:   return launch2<0, 0, EPI_COMBINE>(ta, tb, ta, tb, p, s);
    case 10:  return launch2<0, 1, EPI_STORE>(ta, tb, ta, tb, p, s);
    case 12:  return launch2<0, 1, EPI_DGELU>(ta, tb, ta, tb, p, s);
    case 15:  return launch2<0, 1, EPI_SCATTER>(ta, tb, ta2, tb2, p, s);
    case 110: return launch2<1, 1, EPI_STORE>(ta, tb, ta, tb, p, s);
    default: break;
  }
  *why = "operand-major / epilogue combination not instantiated";
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------- SIMT reference
namespace {
__global__ void gemm_ref_kernel(GemmArgs a) {
  __shared__ float As[16][17];
  __shared__ float Bs[16][17];
  const int b = blockIdx.z;
  const int m = blockIdx.y * 16 + threadIdx.y;
  const int n = blockIdx.x * 16 + threadIdx.x;
  const bf16* A = static_cast<const bf16*>(a.A) + (size_t)b * a.M * a.K;
  const bf16* B = static_cast<const bf16*>(a.B) + (size_t)b * a.N * a.K;
  float acc = 0.f;
  for (int k0 = 0; k0 < a.K; k0 += 16) {
    const int am = blockIdx.y * 16 + threadIdx.y, ak = k0 + threadIdx.x;
    As[threadIdx.y][threadIdx.x] =
        (am < a.M && ak < a.K)
            ? __bfloat162float(a.a_mn ? A[(size_t)ak * a.M + am] : A[(size_t)am * a.K + ak])
            : 0.f;
    const int bn = blockIdx.x * 16 + threadIdx.y, bk = k0 + threadIdx.x;
    Bs[threadIdx.y][threadIdx.x] =
        (bn < a.N && bk < a.K)
            ? __bfloat162float(a.b_mn ? B[(size_t)bk * a.N + bn] : B[(size_t)bn * a.K + bk])
            : 0.f;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += As[threadIdx.y][k] * Bs[threadIdx.x][k];
    __syncthreads();
  }
  if (m < a.M && n < a.N) {
    const size_t o = ((size_t)b * a.M + m) * a.N + n;
    bf16* D = static_cast<bf16*>(a.D);
    bf16* X = static_cast<bf16*>(a.aux);
    if (a.epilogue == EPI_DGELU) acc *= __bfloat162float(X[o]);
    D[o] = __float2bfloat16_rn(a.epilogue == EPI_GELU ? gelu_grad_f(acc) : acc);
    if (a.epilogue == EPI_GELU) X[o] = __float2bfloat16_rn(gelu_f(acc));
  }
}
}  // namespace

cudaError_t gemm_ref(const GemmArgs& a, cudaStream_t s) {
  if (a.batch <= 0 || a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaSuccess;
  dim3 grid((a.N + 15) / 16, (a.M + 15) / 16, a.batch);
  gemm_ref_kernel<<<grid, dim3(16, 16), 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace moe
