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

// Cross-rank barrier over peer memory: thread r stores `epoch` into rank r's flag
// slot for this rank (release, system scope), then acquire-spins until rank r has
// stored `epoch` into ours. Launched after the copy kernel it publishes (stream
// order), so every write of that kernel precedes the flag.
__global__ void peer_barrier_kernel(void* const* __restrict__ table, int nwin, int win, int world,
                                    int rank, uint32_t epoch) {
  const int r = threadIdx.x;
  if (r >= world) return;
  uint32_t* remote = static_cast<uint32_t*>(table[(size_t)r * nwin + win]);
  uint32_t* mine = static_cast<uint32_t*>(table[(size_t)rank * nwin + win]);
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote + rank), "r"(epoch) : "memory");
  uint32_t v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + r) : "memory");
  } while ((int32_t)(v - epoch) < 0);
}

}  // namespace

cudaError_t peer_barrier(void* const* d_table, int nwin, int win, int world, int rank,
                         uint32_t epoch, cudaStream_t s) {
  peer_barrier_kernel<<<1, 32 * ((world + 31) / 32), 0, s>>>(d_table, nwin, win, world, rank, epoch);
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
