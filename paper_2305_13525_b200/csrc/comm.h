// comm.h — the communicator shared by every layer context of a process (moe_comm):
// the peer-visible windows of the exchange, the ring of forward windows, the
// publication primitives (barrier, one-sided readiness signals) and the transport
// behind them.
//
// Transports:
//   IPC   one process per GPU; windows cudaMalloc'd and CUDA-IPC mapped on every rank
//         (handles exchanged once over a temporary NCCL communicator); barriers and
//         signals are release/acquire flags in peer memory with a device deadline.
//   EMU   W ranks emulated in ONE process on ONE device (moe_emu_group, for driving
//         the exchange kernels of any (G_t, G_ep) on a single GPU): every rank's
//         windows are plain allocations on that device and every rank runs the same
//         host code on its own host thread and stream; a barrier is a host barrier
//         plus cudaStreamWaitEvent on every rank's event, a signal is an event. No
//         kernel ever waits on another kernel.
//   NCCL  MOE_F_NCCL_EXCHANGE: no windows; TP / EP communicators split from a world
//         communicator carry the collectives (the library baseline).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/moe.h"
#include "internal.h"
#include "plan.h"

namespace moe {

enum Transport { TR_NONE = 0, TR_IPC = 1, TR_EMU = 2 };

// Window sizes a set of layer configs needs on one rank (all multiples of 2 MiB,
// the allocation granularity, so the plan equals the device memory taken).
struct CommPlan {
  int world = 1, rank = 0, Gt = 1, Gep = 1;
  int depth = 2;                 // ring slots of (X, O)
  int64_t timeout_ms = 60000;    // deadline of every barrier / signal wait
  bool peer = false;             // any config uses the peer-memory exchange
  bool nccl = false;             // any config uses MOE_F_NCCL_EXCHANGE
  bool nvls = false;             // any config uses MOE_F_NVLS (multicast region)
  size_t expert_space = 0, slot_space = 0, tp_space = 0;
  size_t flags_bytes = 0, meta_bytes = 0;
  size_t total = 0;              // device bytes moe_comm_create allocates
};

moe_status make_comm_plan(const moe_config* cfgs, int n, int world, int rank, CommPlan* p,
                          std::string* why);

// MOE_F_NVLS (nvls.cpp): the windows DTD's all-gathers write (X / O rings, dY, dS) live in one
// VMM region per rank, mapped by every peer (fabric handles) and bound to the TP group's
// multicast object, mapped at mcva: a multimem.st at mcva + off reaches off in every TP
// member's region.
struct NvlsRegion {
  size_t size = 0;
  int dev = 0;
  CUmemGenericAllocationHandle phys = 0, mc = 0;
  bool have_phys = false, have_mc = false, bound = false;
  int own_fds[2] = {-1, -1};   // exported descriptors, closed once every peer imported them
  void* uc = nullptr;     // this rank's region
  void* mcva = nullptr;   // the TP group's multicast mapping
  std::vector<void*> peer_uc;  // [world] every rank's region, mapped here
  std::vector<CUmemGenericAllocationHandle> imported;
};
moe_status nvls_create(NvlsRegion* r, size_t bytes, int world, int rank, int Gt, ncclComm_t comm,
                       std::string* why);
void nvls_destroy(NvlsRegion* r);

constexpr int SIG_OFF = 4096;    // byte offset of the signal slots in the flag window
constexpr int PIECE_ARENA = 1 << 16;  // Piece entries in the comm's metadata block

}  // namespace moe

struct moe_emu_group;

struct moe_comm {
  moe::CommPlan plan;
  moe::Transport tr = moe::TR_NONE;
  // window ids: fixed ones, then the X ring, then the O ring
  enum { W_DY = 0, W_DS = 1, W_FLAGS = 2, W_Y = 3, W_DXP = 4, W_RING = 5 };
  int nwin = 0;
  int wx(int s) const { return W_RING + s; }
  int wo(int s) const { return W_RING + plan.depth + s; }
  std::vector<void*> win;        // this rank's windows [nwin]
  std::vector<void*> mcwin;      // [nwin] multicast mapping of a window (MOE_F_NVLS, IPC), else null
  std::vector<size_t> region_off;  // [nwin] offset in the NVLS region, or SIZE_MAX
  moe::NvlsRegion nvls;
  std::vector<void*> opened;     // IPC mappings of the peers' windows
  std::vector<void*> h_table;    // [world][nwin]
  void** d_table = nullptr;      // device copy of h_table (in meta)
  uint8_t* meta = nullptr;       // one allocation: d_table, the piece arena
  moe::Piece* arena = nullptr;
  int arena_used = 0;
  ncclComm_t world_comm = nullptr, tp_comm = nullptr, ep_comm = nullptr;
  moe_emu_group* emu = nullptr;
  int32_t* err_host = nullptr;   // host-mapped error word (device deadline failures)
  int32_t* err_dev = nullptr;
  uint32_t epoch = 0;            // barrier epoch
  uint32_t sig_epoch = 0;        // readiness-signal epoch
  uint64_t gen = 0;              // forwards that claimed a ring slot
  std::vector<uint64_t> ring_gen;  // generation owning each ring slot
  int refs = 0;                  // layer contexts attached
  bool private_to_ctx = false;   // created by moe_create (destroyed with its ctx)
  bool broken = false;
};

namespace moe {

// Creates / destroys a communicator (collective over the world, or over the emulated group).
moe_status comm_create(const moe_config* cfgs, int n, const uint8_t* uid, moe_emu_group* emu, int world,
                       int rank, moe_comm** out, std::string* why);
void comm_destroy(moe_comm* m);
// A device failure (deadline) recorded by a barrier / wait kernel, or a broken emulated
// group: returns MOE_ERR_TIMEOUT with *why set, else MOE_OK. Does not synchronize.
moe_status comm_check(moe_comm* m, std::string* why);
// Every rank's work enqueued on its stream before the barrier precedes every rank's work
// after it (stream order; no host synchronization in the IPC transport).
moe_status comm_barrier(moe_comm* m, cudaStream_t st, std::string* why);
// One-sided readiness: after this stream's prior work, tell rank `dst` that exchange
// `epoch` of this rank is in its window; comm_wait makes `st` wait for that signal of `src`.
moe_status comm_signal(moe_comm* m, int dst, uint32_t epoch, cudaStream_t st, std::string* why);
moe_status comm_wait(moe_comm* m, int src, uint32_t epoch, cudaStream_t st, std::string* why);
int emu_world(const moe_emu_group* g);
// Piece storage for a context's exchange lists (device memory inside the comm's metadata).
Piece* comm_pieces(moe_comm* m, int n);

}  // namespace moe
