// peer.cu — the expert-parallel exchange over NVLink peer memory.
//
// F4+F5 / B2+B3 ("dispatch": slot space -> expert space) and F9+F10 / B8+B9
// ("return": expert space -> slot space) as ONE copy kernel per exchange: every
// contiguous C_s x H piece is written by this rank straight into the destination
// rank's window (CUDA-IPC mapped, reached through NVSwitch), including the pieces
// DTD's all-gather would otherwise re-send (the all-gather is folded into the
// same writes). NCCL P2P on this box peaks near 250 GB/s per rank and degrades
// with the number of pieces; direct 16-byte peer stores run at link speed.
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int XC_THREADS = 256;
constexpr int XC_CHUNK = XC_THREADS * 16 * 8;  // bytes per block: 8 x 16 B per thread

__global__ void __launch_bounds__(XC_THREADS)
    exchange_kernel(const uint8_t* __restrict__ src, void* const* __restrict__ table, int nwin,
                    int win, const Piece* __restrict__ pieces, size_t piece_bytes,
                    int chunks_per_piece) {
  const int pi = blockIdx.x / chunks_per_piece;
  const int ci = blockIdx.x % chunks_per_piece;
  const Piece pc = pieces[pi];
  uint8_t* dst = static_cast<uint8_t*>(table[(size_t)pc.dst_rank * nwin + win]) + pc.dst_off;
  const uint8_t* s = src + pc.src_off;
  const size_t base = (size_t)ci * XC_CHUNK;
  uint4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const size_t o = base + ((size_t)k * XC_THREADS + threadIdx.x) * 16;
    v[k] = o < piece_bytes ? ld_nc_v4(s + o) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const size_t o = base + ((size_t)k * XC_THREADS + threadIdx.x) * 16;
    if (o < piece_bytes) st_v4(dst + o, v[k]);
  }
  __threadfence_system();
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bounded acquire-spin until *flag >= epoch (wrap-safe). Gives up after timeout_ns and
// records `code` in the host-mapped error word, which the next library call reports
// (MOE_ERR_TIMEOUT); once the word is set no later wait spins at all, so a dead or
// absent rank costs one deadline, not one per barrier.
__device__ __forceinline__ bool bounded_wait(const uint32_t* flag, uint32_t epoch, int32_t* err,
                                             uint64_t timeout_ns, int32_t code) {
  if (*reinterpret_cast<volatile int32_t*>(err) != 0) return false;
  const uint64_t t0 = globaltimer_ns();
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int32_t)(v - epoch) >= 0) return true;
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicCAS(err, 0, code);
      __threadfence_system();
      return false;
    }
    __nanosleep(100);
  }
}

// Cross-rank barrier over peer memory: thread r stores `epoch` into rank r's flag
// slot for this rank (release, system scope), then acquire-spins (bounded) until rank r
// has stored `epoch` into ours. Launched after the copy kernel it publishes (stream
// order), so every write of that kernel precedes the flag.
__global__ void peer_barrier_kernel(void* const* __restrict__ table, int nwin, int win, int world,
                                    int rank, uint32_t epoch, int32_t* err, uint64_t timeout_ns) {
  const int r = threadIdx.x;
  if (r >= world) return;
  uint32_t* remote = static_cast<uint32_t*>(table[(size_t)r * nwin + win]);
  uint32_t* mine = static_cast<uint32_t*>(table[(size_t)rank * nwin + win]);
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote + rank), "r"(epoch) : "memory");
  bounded_wait(mine + r, epoch, err, timeout_ns, 1);
}

// Fused TP reduction + return exchange (F8-F10 / B7-B9 for G_t > 1): one warp per
// expert-space row of the slices this rank reduces (DTD: its own slot slice t; vanilla:
// all slices), summing the G_t partials of the TP group in fixed order t' = 0..G_t-1 in
// fp32 (partners' windows read over NVLink), rounding once to bf16 and storing the row
// into the slot-space window of the source rank(s): every TP rank of the source under
// DTD (the folded all-gather), the same-t rank under vanilla. With G_t = 2 this equals
// NCCL's bf16 sum bit for bit.
constexpr int RR_WARPS = 8;
__global__ void __launch_bounds__(RR_WARPS * 32)
    reduce_return_kernel(ReduceReturn rr, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * RR_WARPS + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int nsl = rr.dtd ? 1 : rr.Gt;  // slices reduced by this rank
  const int64_t cs = r % rr.Cs;
  int64_t q = r / rr.Cs;
  const int src = (int)(q % rr.Gep);
  q /= rr.Gep;
  const int tt = rr.dtd ? rr.t : (int)(q % nsl);
  const int el = (int)(q / nsl);
  const size_t rowb = (size_t)rr.H * 2;
  const size_t xoff = ((((size_t)el * rr.Gt + tt) * rr.Gep + src) * rr.Cs + cs) * rowb;
  const int e = rr.ep * rr.El + el;
  const size_t ooff = (((size_t)tt * rr.E + e) * rr.Cs + cs) * rowb;
  const int nv = rr.H / 8;
  const int tp0 = (rr.d * rr.Gep + rr.ep) * rr.Gt;
  const int dst0 = (rr.d * rr.Gep + src) * rr.Gt;
  constexpr int U = 4;
  for (int v0 = 0; v0 < nv; v0 += 32 * U) {
    float acc[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[u][k] = 0.f;
    for (int tp = 0; tp < rr.Gt; ++tp) {
      const uint8_t* base = static_cast<const uint8_t*>(rr.table[(size_t)(tp0 + tp) * rr.nwin + rr.src_win]) + xoff;
      uint4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32 + lane;
        b[u] = v < nv ? ld_nc_v4(base + (size_t)v * 16) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = unpack_bf16x2(w[k]);
          acc[u][2 * k] += f.x;
          acc[u][2 * k + 1] += f.y;
        }
      }
    }
    uint4 o[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      o[u] = make_uint4(pack_bf16x2(acc[u][0], acc[u][1]), pack_bf16x2(acc[u][2], acc[u][3]),
                        pack_bf16x2(acc[u][4], acc[u][5]), pack_bf16x2(acc[u][6], acc[u][7]));
    const bool mc = rr.fold && rr.mc && src == rr.ep;  // own group: one multicast store
    const int nd = mc ? 1 : (rr.fold ? rr.Gt : 1);
    for (int k = 0; k < nd; ++k) {
      const int dr = dst0 + (rr.fold ? k : rr.t);
      uint8_t* dst = mc ? static_cast<uint8_t*>(rr.mc) + ooff
                        : static_cast<uint8_t*>(rr.table[(size_t)dr * rr.nwin + rr.dst_win]) + ooff;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nv) {
          if (mc) st_mc_v4(dst + (size_t)v * 16, o[u]);
          else st_v4(dst + (size_t)v * 16, o[u]);
        }
      }
    }
  }
  __threadfence_system();
}

// DTD all-gather within the TP group (MOE_F_NVLS): nseg segments of seg_bytes at
// base_off + i * stride of window `win` of this rank go to the same offsets of every TP
// rank's window — through the TP group's multicast mapping `mc` (one multimem.st,
// replicated by NVSwitch: the sender's egress is the slice once whatever G_t), or, with
// no multicast mapping (emulated ranks), one unicast store per TP peer. Bytes are copied
// as 16-byte vectors, bit for bit.
__global__ void __launch_bounds__(256)
    tp_allgather_kernel(TpAllGather ag) {
  const uint64_t nv = ag.seg_bytes / 16;
  const uint64_t total = nv * (uint64_t)ag.nseg;
  const uint8_t* src = static_cast<const uint8_t*>(ag.table[(size_t)ag.rank * ag.nwin + ag.win]);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t seg = i / nv, v = i - seg * nv;
    const uint64_t off = ag.base_off + seg * ag.stride + v * 16;
    const uint4 x = ld_nc_v4(src + off);
    if (ag.mc) {
      st_mc_v4(static_cast<uint8_t*>(ag.mc) + off, x);
    } else {
      for (int tp = 0; tp < ag.Gt; ++tp) {
        const int r = ag.tp0 + tp;
        if (r == ag.rank) continue;
        st_v4(static_cast<uint8_t*>(ag.table[(size_t)r * ag.nwin + ag.win]) + off, x);
      }
    }
  }
  __threadfence_system();
}

// Point-to-point readiness flags (per-source pipelining of the split exchange): the
// source stores `epoch` (release, system scope) into slot `src` of the destination's
// flag region after its copies to that destination; the destination's stream spins
// (acquire) on that slot before the GEMM over that source's rows.
__global__ void peer_signal_kernel(uint32_t* flag, uint32_t epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

__global__ void peer_wait_kernel(const uint32_t* flag, uint32_t epoch, int32_t* err, uint64_t timeout_ns) {
  bounded_wait(flag, epoch, err, timeout_ns, 2);
}

}  // namespace

cudaError_t tp_allgather(const TpAllGather& ag, cudaStream_t s) {
  const uint64_t total = ag.seg_bytes / 16 * (uint64_t)ag.nseg;
  if (!total) return cudaSuccess;
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;  // grid-stride: a few waves of 256-thread CTAs
  tp_allgather_kernel<<<(unsigned)blocks, 256, 0, s>>>(ag);
  return cudaGetLastError();
}

cudaError_t peer_signal(uint32_t* flag, uint32_t epoch, cudaStream_t s) {
  peer_signal_kernel<<<1, 1, 0, s>>>(flag, epoch);
  return cudaGetLastError();
}

cudaError_t peer_wait(const uint32_t* flag, uint32_t epoch, int32_t* err, uint64_t timeout_ns,
                      cudaStream_t s) {
  peer_wait_kernel<<<1, 1, 0, s>>>(flag, epoch, err, timeout_ns);
  return cudaGetLastError();
}

cudaError_t reduce_return(const ReduceReturn& rr, cudaStream_t s) {
  const int64_t rows = (int64_t)rr.El * rr.Gep * rr.Cs * (rr.dtd ? 1 : rr.Gt);
  if (rows <= 0) return cudaSuccess;
  reduce_return_kernel<<<(unsigned)((rows + RR_WARPS - 1) / RR_WARPS), RR_WARPS * 32, 0, s>>>(rr, rows);
  return cudaGetLastError();
}

cudaError_t peer_barrier(void* const* d_table, int nwin, int win, int world, int rank,
                         uint32_t epoch, int32_t* err, uint64_t timeout_ns, cudaStream_t s) {
  peer_barrier_kernel<<<1, 32 * ((world + 31) / 32), 0, s>>>(d_table, nwin, win, world, rank, epoch, err,
                                                              timeout_ns);
  return cudaGetLastError();
}

cudaError_t peer_exchange(const void* src, void* const* d_table, int nwin, int win,
                          const Piece* d_pieces, int npieces, size_t piece_bytes, cudaStream_t s) {
  if (npieces <= 0 || piece_bytes == 0) return cudaSuccess;
  const int cpp = (int)((piece_bytes + XC_CHUNK - 1) / XC_CHUNK);
  exchange_kernel<<<(unsigned)((int64_t)npieces * cpp), XC_THREADS, 0, s>>>(
      static_cast<const uint8_t*>(src), d_table, nwin, win, d_pieces, piece_bytes, cpp);
  return cudaGetLastError();
}

}  // namespace moe
