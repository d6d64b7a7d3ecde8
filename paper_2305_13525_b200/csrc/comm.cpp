// comm.cpp — moe_comm: windows, ring slots, barrier / signal transports (comm.h).
#include "comm.h"

#include <algorithm>
#include <climits>
#include <cstdint>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

// W ranks emulated in one process on one device (include/moe.h, moe_emu_group_create).
struct moe_emu_group {
  int world = 0;
  int device = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  int phase_kind = -1;                   // what the ranks of the current phase are doing
  bool broken = false;
  std::vector<std::vector<void*>> wins;  // [rank] -> that rank's windows
  std::vector<cudaEvent_t> bar_ev;       // [2][world]: barrier epochs by parity
  std::vector<cudaEvent_t> sig_ev;       // [2][world (src)][world (dst)]
  std::vector<uint32_t> sig_val;         // [src][dst]: last signalled epoch
};

namespace moe {
namespace {

constexpr size_t GRAN = (size_t)2 << 20;  // cudaMalloc granularity of large allocations
size_t round_gran(size_t b) { return b == 0 ? 0 : (b + GRAN - 1) / GRAN * GRAN; }

// Host barrier of the emulated group; false on timeout or when ranks arrive for different
// things (a layer call vs create / destroy: out of step) — the group is then broken for good.
enum { BAR_CALL = 0, BAR_CREATE = 1, BAR_DESTROY = 2 };
bool host_barrier(moe_emu_group* g, int64_t timeout_ms, int kind) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) return false;
  const uint64_t ph = g->phase;
  if (g->arrived == 0) g->phase_kind = kind;
  if (g->phase_kind != kind) {
    g->broken = true;
    g->cv.notify_all();
    return false;
  }
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->phase;
    g->cv.notify_all();
    return true;
  }
  const bool ok = g->cv.wait_for(lk, std::chrono::milliseconds(timeout_ms),
                                 [&] { return g->phase != ph || g->broken; });
  if (!ok) {
    g->broken = true;
    g->cv.notify_all();
  }
  return ok && !g->broken;
}

moe_status cuda_fail(cudaError_t e, const char* what, std::string* why) {
  *why = std::string(what) + ": " + cudaGetErrorString(e);
  return MOE_ERR_CUDA;
}

#define CT(expr)                                          \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr, why); \
  } while (0)

}  // namespace

moe_status make_comm_plan(const moe_config* cfgs, int n, int world, int rank, CommPlan* p, std::string* why) {
  if (!cfgs || n < 1 || !p) { *why = "need at least one layer config"; return MOE_ERR_ARG; }
  CommPlan q;
  q.world = world;
  q.rank = rank;
  q.depth = 0;
  q.timeout_ms = 0;
  for (int i = 0; i < n; ++i) {
    Dims d;
    moe_status s = make_dims(&cfgs[i], world, rank, &d, why);
    if (s != MOE_OK) return s;
    if (i == 0) { q.Gt = d.Gt; q.Gep = d.Gep; }
    if (d.Gt != q.Gt || d.Gep != q.Gep) {
      *why = "every layer of a communicator needs the same g_tensor and g_expert";
      return MOE_ERR_ARG;
    }
    q.peer |= d.peer;
    q.nccl |= world > 1 && !d.peer;
    q.nvls |= d.nvls;
    q.expert_space = std::max(q.expert_space, (size_t)d.El * d.R * d.H * 2);
    q.slot_space = std::max(q.slot_space, (size_t)d.E * d.C * d.H * 2);
    if (d.Gt > 1) q.tp_space = std::max(q.tp_space, (size_t)d.El * d.R * d.H * 2);
    q.depth = std::max(q.depth, d.ring_depth);
    q.timeout_ms = std::max<int64_t>(q.timeout_ms, d.timeout_ms);
  }
  if (q.peer) {
    const int nwin = moe_comm::W_RING + 2 * q.depth;
    q.flags_bytes = SIG_OFF + 4 * (size_t)world;
    q.meta_bytes = sizeof(void*) * (size_t)world * nwin + sizeof(Piece) * (size_t)PIECE_ARENA;
    q.total = round_gran(q.expert_space) * (q.depth + 1)      // X ring + dY
              + round_gran(q.slot_space) * (q.depth + 1)      // O ring + dS
              + round_gran(q.tp_space) * 2                    // Y, dXp (TP partials)
              + round_gran(q.flags_bytes) + round_gran(q.meta_bytes);
  }
  *p = q;
  return MOE_OK;
}

moe_status comm_create(const moe_config* cfgs, int n, const uint8_t* uid, moe_emu_group* emu, int world,
                       int rank, moe_comm** out, std::string* why) {
  *out = nullptr;
  CommPlan plan;
  moe_status s = make_comm_plan(cfgs, n, world, rank, &plan, why);
  if (s != MOE_OK) return s;
  if (emu) {
    if (emu->world != world) { *why = "emulated group size != world"; return MOE_ERR_ARG; }
    if (plan.nccl) { *why = "MOE_F_NCCL_EXCHANGE cannot be emulated on one device"; return MOE_ERR_UNSUPPORTED; }
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != emu->device) { *why = "emulated ranks must run on the group's device"; return MOE_ERR_ARG; }
  } else if (world > 1 && !uid) {
    *why = "uid required when world > 1";
    return MOE_ERR_ARG;
  }
  moe_comm* m = new moe_comm();
  m->plan = plan;
  m->emu = emu;
  m->tr = !plan.peer ? TR_NONE : (emu ? TR_EMU : TR_IPC);
  auto bail = [&](moe_status st) {
    comm_destroy(m);
    return st;
  };
#define CB(expr)                                                   \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return bail(cuda_fail(_e, #expr, why)); \
  } while (0)
  size_t region = 0;  // bytes of the NVLS multicast region (MOE_F_NVLS over IPC)
  CB(cudaHostAlloc(reinterpret_cast<void**>(&m->err_host), sizeof(int32_t), cudaHostAllocMapped));
  *m->err_host = 0;
  CB(cudaHostGetDevicePointer(reinterpret_cast<void**>(&m->err_dev), m->err_host, 0));
  if (plan.peer) {
    m->nwin = moe_comm::W_RING + 2 * plan.depth;
    m->win.assign(m->nwin, nullptr);
    m->ring_gen.assign(plan.depth, 0);
    std::vector<size_t> sz(m->nwin, 0);
    sz[moe_comm::W_DY] = plan.expert_space;
    sz[moe_comm::W_DS] = plan.slot_space;
    sz[moe_comm::W_FLAGS] = plan.flags_bytes;
    sz[moe_comm::W_Y] = plan.tp_space;
    sz[moe_comm::W_DXP] = plan.tp_space;
    for (int r = 0; r < plan.depth; ++r) {
      sz[m->wx(r)] = plan.expert_space;
      sz[m->wo(r)] = plan.slot_space;
    }
    // MOE_F_NVLS over IPC: the X / O rings, dY and dS live in the multicast region (created
    // once the world communicator exists, below); everything else is cudaMalloc'd
    m->mcwin.assign(m->nwin, nullptr);
    m->region_off.assign(m->nwin, SIZE_MAX);
    if (plan.nvls && !emu && world > 1) {
      for (int w = 0; w < m->nwin; ++w) {
        const bool in = w == moe_comm::W_DY || w == moe_comm::W_DS || w >= moe_comm::W_RING;
        if (!in || !sz[w]) continue;
        m->region_off[w] = region;
        region += round_gran(sz[w]);
      }
    }
    for (int w = 0; w < m->nwin; ++w) {
      if (!sz[w] || m->region_off[w] != SIZE_MAX) continue;
      CB(cudaMalloc(&m->win[w], round_gran(sz[w])));
      CB(cudaMemset(m->win[w], 0, round_gran(sz[w])));
    }
    CB(cudaMalloc(&m->meta, round_gran(plan.meta_bytes)));
    m->d_table = reinterpret_cast<void**>(m->meta);
    m->arena = reinterpret_cast<Piece*>(m->meta + sizeof(void*) * (size_t)world * m->nwin);
    m->h_table.assign((size_t)world * m->nwin, nullptr);
  }
  if (m->tr == TR_EMU) {
    {
      std::lock_guard<std::mutex> lk(emu->mu);
      emu->wins[rank] = m->win;
    }
    if (!host_barrier(emu, plan.timeout_ms, BAR_CREATE)) {
      *why = "emulated ranks did not all join within the deadline";
      return bail(MOE_ERR_TIMEOUT);
    }
    for (int r = 0; r < world; ++r)
      for (int w = 0; w < m->nwin; ++w) m->h_table[(size_t)r * m->nwin + w] = emu->wins[r][w];
  } else if (world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&m->world_comm, world, id, rank);
    if (r != ncclSuccess) {
      *why = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      m->world_comm = nullptr;
      return bail(MOE_ERR_NCCL);
    }
    if (region) {
      s = nvls_create(&m->nvls, region, world, rank, plan.Gt, m->world_comm, why);
      if (s != MOE_OK) return bail(s);
      for (int w = 0; w < m->nwin; ++w)
        if (m->region_off[w] != SIZE_MAX) {
          m->win[w] = static_cast<uint8_t*>(m->nvls.uc) + m->region_off[w];
          m->mcwin[w] = static_cast<uint8_t*>(m->nvls.mcva) + m->region_off[w];
        }
    }
    if (plan.peer) {
      // exchange the IPC handles of every window once over the world communicator
      const int nw = m->nwin;
      std::vector<cudaIpcMemHandle_t> mine(nw);
      std::memset(mine.data(), 0, sizeof(cudaIpcMemHandle_t) * nw);
      for (int w = 0; w < nw; ++w)
        if (m->win[w] && m->region_off[w] == SIZE_MAX) CB(cudaIpcGetMemHandle(&mine[w], m->win[w]));
      const size_t hb = sizeof(cudaIpcMemHandle_t) * nw;
      uint8_t* dbuf = nullptr;
      CB(cudaMalloc(&dbuf, hb * world));
      cudaStream_t st = nullptr;
      cudaError_t e = cudaMemcpy(dbuf + hb * rank, mine.data(), hb, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      if (e != cudaSuccess) { cudaFree(dbuf); return bail(cuda_fail(e, "handle staging", why)); }
      r = ncclAllGather(dbuf + hb * rank, dbuf, hb, ncclUint8, m->world_comm, st);
      if (r == ncclSuccess) e = cudaStreamSynchronize(st);
      std::vector<cudaIpcMemHandle_t> all((size_t)nw * world);
      if (r == ncclSuccess && e == cudaSuccess) e = cudaMemcpy(all.data(), dbuf, hb * world, cudaMemcpyDeviceToHost);
      cudaStreamDestroy(st);
      cudaFree(dbuf);
      if (r != ncclSuccess) { *why = std::string("ncclAllGather: ") + ncclGetErrorString(r); return bail(MOE_ERR_NCCL); }
      if (e != cudaSuccess) return bail(cuda_fail(e, "handle exchange", why));
      for (int q = 0; q < world; ++q)
        for (int w = 0; w < nw; ++w) {
          void*& slot = m->h_table[(size_t)q * nw + w];
          if (q == rank) { slot = m->win[w]; continue; }
          if (!m->win[w]) continue;  // same plan on every rank: absent everywhere
          if (m->region_off[w] != SIZE_MAX) {  // NVLS region: the peer's fabric-handle mapping
            slot = static_cast<uint8_t*>(m->nvls.peer_uc[q]) + m->region_off[w];
            continue;
          }
          CB(cudaIpcOpenMemHandle(&slot, all[(size_t)q * nw + w], cudaIpcMemLazyEnablePeerAccess));
          m->opened.push_back(slot);
        }
    }
    if (plan.nccl) {
      const int Gt = plan.Gt, Gep = plan.Gep;
      const int t = rank % Gt, ep = (rank / Gt) % Gep, dd = rank / (Gt * Gep);
      r = ncclCommSplit(m->world_comm, dd * Gep + ep, t, &m->tp_comm, nullptr);
      if (r == ncclSuccess) r = ncclCommSplit(m->world_comm, dd * Gt + t, ep, &m->ep_comm, nullptr);
      if (r != ncclSuccess) {
        *why = std::string("ncclCommSplit: ") + ncclGetErrorString(r);
        return bail(MOE_ERR_NCCL);
      }
    } else {
      // peer mode needs no NCCL after the handle exchange: release its buffers
      ncclCommDestroy(m->world_comm);
      m->world_comm = nullptr;
    }
  }
  if (plan.peer)
    CB(cudaMemcpy(m->d_table, m->h_table.data(), sizeof(void*) * m->h_table.size(), cudaMemcpyHostToDevice));
#undef CB
  *out = m;
  return MOE_OK;
}

void comm_destroy(moe_comm* m) {
  if (!m) return;
  if (m->tr == TR_EMU && m->emu) host_barrier(m->emu, 10000, BAR_DESTROY);  // no rank frees while a peer may write
  for (void* p : m->opened) cudaIpcCloseMemHandle(p);
  for (size_t w = 0; w < m->win.size(); ++w)
    if (m->win[w] && (m->region_off.empty() || m->region_off[w] == SIZE_MAX)) cudaFree(m->win[w]);
  if (m->nvls.size) {
    cudaDeviceSynchronize();  // no exchange may still be writing the region
    nvls_destroy(&m->nvls);
  }
  if (m->meta) cudaFree(m->meta);
  if (m->err_host) cudaFreeHost(m->err_host);
  if (m->tp_comm) ncclCommDestroy(m->tp_comm);
  if (m->ep_comm) ncclCommDestroy(m->ep_comm);
  if (m->world_comm) ncclCommDestroy(m->world_comm);
  delete m;
}

moe_status comm_check(moe_comm* m, std::string* why) {
  if (!m) return MOE_OK;
  const int32_t e = m->err_host ? *reinterpret_cast<volatile int32_t*>(m->err_host) : 0;
  if (e) {
    *why = e == 1 ? "a peer rank did not reach a window barrier within the deadline"
                  : "a peer rank's readiness signal did not arrive within the deadline";
    m->broken = true;
    return MOE_ERR_TIMEOUT;
  }
  if (m->tr == TR_EMU) {
    std::lock_guard<std::mutex> lk(m->emu->mu);
    if (m->emu->broken) {
      *why = "an emulated rank did not reach a barrier within the deadline";
      m->broken = true;
      return MOE_ERR_TIMEOUT;
    }
  }
  if (m->broken) { *why = "communicator broken by an earlier deadline failure"; return MOE_ERR_TIMEOUT; }
  return MOE_OK;
}

moe_status comm_barrier(moe_comm* m, cudaStream_t st, std::string* why) {
  const int world = m->plan.world, rank = m->plan.rank;
  const uint32_t ep = ++m->epoch;
  if (m->tr == TR_IPC) {
    const uint64_t tns = (uint64_t)m->plan.timeout_ms * 1000000ull;
    CT(peer_barrier(m->d_table, m->nwin, moe_comm::W_FLAGS, world, rank, ep, m->err_dev, tns, st));
    return MOE_OK;
  }
  moe_emu_group* g = m->emu;
  cudaEvent_t* ev = &g->bar_ev[(size_t)(ep & 1) * world];
  CT(cudaEventRecord(ev[rank], st));
  if (!host_barrier(g, m->plan.timeout_ms, BAR_CALL)) {
    m->broken = true;
    *why = "an emulated rank did not reach the barrier within the deadline (absent or out of step)";
    return MOE_ERR_TIMEOUT;
  }
  for (int r = 0; r < world; ++r)
    if (r != rank) CT(cudaStreamWaitEvent(st, ev[r], 0));
  return MOE_OK;
}

moe_status comm_signal(moe_comm* m, int dst, uint32_t epoch, cudaStream_t st, std::string* why) {
  const int world = m->plan.world, rank = m->plan.rank;
  if (m->tr == TR_IPC) {
    uint32_t* flag = reinterpret_cast<uint32_t*>(
        static_cast<uint8_t*>(m->h_table[(size_t)dst * m->nwin + moe_comm::W_FLAGS]) + SIG_OFF) + rank;
    CT(peer_signal(flag, epoch, st));
    return MOE_OK;
  }
  moe_emu_group* g = m->emu;
  CT(cudaEventRecord(g->sig_ev[((size_t)(epoch & 1) * world + rank) * world + dst], st));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->sig_val[(size_t)rank * world + dst] = epoch;
  }
  g->cv.notify_all();
  return MOE_OK;
}

moe_status comm_wait(moe_comm* m, int src, uint32_t epoch, cudaStream_t st, std::string* why) {
  const int world = m->plan.world, rank = m->plan.rank;
  if (m->tr == TR_IPC) {
    const uint32_t* flag = reinterpret_cast<const uint32_t*>(
        static_cast<uint8_t*>(m->win[moe_comm::W_FLAGS]) + SIG_OFF) + src;
    CT(peer_wait(flag, epoch, m->err_dev, (uint64_t)m->plan.timeout_ms * 1000000ull, st));
    return MOE_OK;
  }
  moe_emu_group* g = m->emu;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    const uint32_t* v = &g->sig_val[(size_t)src * world + rank];
    const bool ok = g->cv.wait_for(lk, std::chrono::milliseconds(m->plan.timeout_ms),
                                   [&] { return (int32_t)(*v - epoch) >= 0 || g->broken; });
    if (!ok || g->broken) {
      g->broken = true;
      g->cv.notify_all();
      m->broken = true;
      *why = "an emulated rank's readiness signal did not arrive within the deadline";
      return MOE_ERR_TIMEOUT;
    }
  }
  CT(cudaStreamWaitEvent(st, g->sig_ev[((size_t)(epoch & 1) * world + src) * world + rank], 0));
  return MOE_OK;
}

int emu_world(const moe_emu_group* g) { return g->world; }

Piece* comm_pieces(moe_comm* m, int n) {
  if (!m->arena || m->arena_used + n > PIECE_ARENA) return nullptr;
  Piece* p = m->arena + m->arena_used;
  m->arena_used += n;
  return p;
}

}  // namespace moe

// ---------------------------------------------------------------- emulated group (C ABI)
extern "C" {

moe_status moe_emu_group_create(int world, moe_emu_group** out) {
  if (!out || world < 1 || world > 1024) return MOE_ERR_ARG;
  *out = nullptr;
  moe_emu_group* g = new moe_emu_group();
  g->world = world;
  if (cudaGetDevice(&g->device) != cudaSuccess) { delete g; return MOE_ERR_CUDA; }
  g->wins.assign(world, {});
  g->bar_ev.assign((size_t)2 * world, nullptr);
  g->sig_ev.assign((size_t)2 * world * world, nullptr);
  g->sig_val.assign((size_t)world * world, 0);
  for (auto* v : {&g->bar_ev, &g->sig_ev})
    for (auto& e : *v)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        moe_emu_group_destroy(g);
        return MOE_ERR_CUDA;
      }
  *out = g;
  return MOE_OK;
}

moe_status moe_emu_group_destroy(moe_emu_group* g) {
  if (!g) return MOE_OK;
  for (auto* v : {&g->bar_ev, &g->sig_ev})
    for (auto e : *v)
      if (e) cudaEventDestroy(e);
  delete g;
  return MOE_OK;
}

}  // extern "C"
