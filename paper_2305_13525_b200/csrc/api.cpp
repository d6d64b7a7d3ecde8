// api.cpp — the C ABI of include/moe.h: context, NCCL communicators, and the
// per-call step list of SURVEY §8(a) enqueued on the caller's stream.
//
// HBM layouts:
//   slot space   [G_t][E][C_s][H]          dispatch send buffer D, combine source O, dO, dS
//   expert space [E_l][G_t][G_ep][C_s][H]  expert inputs X, Ypart, dY, dXpart (R = G_ep*C rows / expert)
// Slot c of expert e sits in slot slice c / C_s, so DTD's "drop"
// is "dispatch only my slice", its all-gather is an in-place
// ncclAllGather per local expert over the TP communicator, and AR + drop on the
// return path is an in-place ncclReduceScatter (R11, R12). Vanilla and
// DTD feed the expert GEMMs the same rows in the same positions.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/moe.h"
#include "../../include/moe_optim.h"
#include "internal.h"
#include "comm.h"

#include <nvtx3/nvToolsExt.h>
#include "plan.h"

using namespace moe;

struct moe_ctx {
  Dims d;
  moe_config cfg;
  SavedLayout sv;
  ScratchLayout sc;
  uint8_t* scratch = nullptr;
  size_t scratch_bytes = 0;
  moe_comm* comm = nullptr;  // world > 1: windows, ring, NCCL communicators (comm.h)
  bool poisoned = false;
  uint64_t priority_seed = 0;  // MOE_F_RANDOM_PRIORITY key (moe_set_priority_seed)
  bool no_fused_dx = false;    // MOE_NO_FUSED_DX=1: B10 as a separate kernel (A/B, tests)
  bool no_fused_combine = false;  // MOE_NO_FUSED_COMBINE=1: F11 as a separate kernel
  bool no_gemm_signal = false;    // MOE_NO_GEMM_SIGNAL=1: GEMM2 parts as separate launches (A/B)
  bool no_fused_return = false;   // MOE_NO_FUSED_RETURN=1: F9 by copy engines after GEMM2 parts (A/B)
  moe_stats stats;
  std::unordered_set<const void*> saved_written;
  // peer-memory exchange (d.peer): this layer's piece lists over the comm's windows
  std::vector<Piece> h_ret;        // return pieces (host copy, for copy-engine exchanges)
  Piece* d_ret_local = nullptr;    // this rank's own return pieces (SM copy kernel; comm arena)
  int n_ret_local = 0;
  std::vector<int> h_ret_el;       // local expert of each return piece
  cudaStream_t side = nullptr;     // copy-engine / overlap stream
  bool overlap = true;             // MOE_NO_OVERLAP=1: serial return exchanges (A/B knob)
  cudaEvent_t ev[4] = {};
  cudaEvent_t evp[4] = {};  // GEMM2 parts (G_t = 1 return overlap)
  // GEMM2 part-completion flags (device, comm arena): cnt[4] then flag[4]; the side stream
  // waits on flag values (cuStreamWaitValue32) instead of part boundaries between launches
  int32_t* gsig = nullptr;
  uint32_t gsig_epoch = 0;
  int64_t disp_bytes[3] = {0, 0, 0}, ret_bytes[3] = {0, 0, 0};  // by Piece::kind
  std::unordered_map<const void*, std::pair<int, uint64_t>> saved_slot;  // saved -> (ring slot, gen)
  const void* replayed = nullptr;  // MOE_F_CHECKPOINT: saved blob whose G/A sit in scratch
  const void* last_saved = nullptr;
  cudaStream_t last_stream = nullptr;
  // MOE_F_TIMING: event pairs per kernel class, resolved in moe_stats_get
  bool timing = false;
  struct Span { int cls; cudaEvent_t a, b; };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  ~moe_ctx() {
    for (auto& s : spans) { cudaEventDestroy(s.a); cudaEventDestroy(s.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

namespace {

thread_local std::string g_detail;

moe_status fail(moe_status s, const std::string& why) {
  g_detail = why;
  return s;
}

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      if (ctx) (ctx)->poisoned = true;                                                       \
      return fail(MOE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));         \
    }                                                                                        \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    ncclResult_t _r = (expr);                                                                \
    if (_r != ncclSuccess) {                                                                 \
      if (ctx) (ctx)->poisoned = true;                                                       \
      return fail(MOE_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));         \
    }                                                                                        \
  } while (0)

cudaEvent_t take_event(moe_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// Counts this library's kernel launches per class and, with MOE_F_TIMING,
// brackets the class's work with CUDA events on the launching stream.
// One kernel class of the path: launch count, CUDA events (MOE_F_TIMING) and an NVTX
// range named after the class (host-side; header-only NVTX3, a no-op without a tool).
const char* const kClassNames[8] = {"moe.route", "moe.dispatch", "moe.gemm", "moe.combine",
                                    "moe.combine_bwd", "moe.gate_bwd", "moe.comm", "moe.xfer"};
struct Scope {
  moe_ctx* c;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Scope(moe_ctx* c_, int cls_, cudaStream_t st_, int kernels) : c(c_), cls(cls_), st(st_) {
    nvtxRangePushA(kClassNames[cls]);
    c->stats.kernel_launches[cls] += kernels;
    if (c->timing && (a = take_event(c)) != nullptr) cudaEventRecord(a, st);
  }
  ~Scope() {
    nvtxRangePop();
    if (!a) return;
    cudaEvent_t b = take_event(c);
    if (!b) { c->pool.push_back(a); return; }
    cudaEventRecord(b, st);
    c->spans.push_back({cls, a, b});
  }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T>
T* at(void* base, size_t off) { return reinterpret_cast<T*>(static_cast<uint8_t*>(base) + off); }
template <typename T>
const T* at(const void* base, size_t off) {
  return reinterpret_cast<const T*>(static_cast<const uint8_t*>(base) + off);
}

SlotSpace slot_space(const Dims& d) {
  SlotSpace s;
  s.C = d.C; s.Cs = d.Cs; s.G_t = d.Gt; s.E = d.E; s.H = d.H; s.K = d.K;
  return s;
}

void ledger(moe_ctx* c, int kind, int pass, int64_t wire) {
  c->stats.calls[kind] += 1;
  c->stats.wire_bytes[kind] += wire;
  if (pass == 0) c->stats.forward_calls += 1;
  else if (pass == 1) c->stats.backward_calls += 1;
  else c->stats.replay_calls += 1;
}

// ---- EP exchange between slot space S and expert space X (F4/F9/B2/B8) ----
// dir 0: S_me(tt, p*E_l+el) -> X_p(el, tt, ep_me);  dir 1: X_me(el, tt, p) -> S_p(tt, ep_me*E_l+el).
moe_status ep_exchange(moe_ctx* c, int dir, int pass, void* S, void* X, int lo, int hi,
                       cudaStream_t st) {
  const Dims& d = c->d;
  const size_t piece = (size_t)d.Cs * d.H;  // elements
  const size_t pbytes = piece * 2;
  auto s_at = [&](int tt, int e) { return at<uint8_t>(S, ((size_t)tt * d.E + e) * pbytes); };
  auto x_at = [&](int el, int tt, int src) {
    return at<uint8_t>(X, (((size_t)el * d.Gt + tt) * d.Gep + src) * pbytes);
  };
  // self pieces: device copies
  for (int el = 0; el < d.El; ++el)
    for (int tt = lo; tt < hi; ++tt) {
      if (dir == 0)
        CUDA_TRY(c, cudaMemcpyAsync(x_at(el, tt, d.ep), s_at(tt, d.ep * d.El + el), pbytes,
                                    cudaMemcpyDeviceToDevice, st));
      else
        CUDA_TRY(c, cudaMemcpyAsync(s_at(tt, d.ep * d.El + el), x_at(el, tt, d.ep), pbytes,
                                    cudaMemcpyDeviceToDevice, st));
    }
  if (d.Gep == 1) return MOE_OK;
  NCCL_TRY(c, ncclGroupStart());
  for (int p = 0; p < d.Gep; ++p) {
    if (p == d.ep) continue;
    for (int el = 0; el < d.El; ++el)
      for (int tt = lo; tt < hi; ++tt) {
        if (dir == 0) {
          NCCL_TRY(c, ncclSend(s_at(tt, p * d.El + el), piece, ncclBfloat16, p, c->comm->ep_comm, st));
          NCCL_TRY(c, ncclRecv(x_at(el, tt, p), piece, ncclBfloat16, p, c->comm->ep_comm, st));
        } else {
          NCCL_TRY(c, ncclSend(x_at(el, tt, p), piece, ncclBfloat16, p, c->comm->ep_comm, st));
          NCCL_TRY(c, ncclRecv(s_at(tt, p * d.El + el), piece, ncclBfloat16, p, c->comm->ep_comm, st));
        }
      }
  }
  NCCL_TRY(c, ncclGroupEnd());
  ledger(c, MOE_COLL_A2A, pass, (int64_t)(d.Gep - 1) * d.El * (hi - lo) * (int64_t)pbytes);
  return MOE_OK;
}

// F5/B3: in-place all-gather of expert space over TP, one call per local expert.
moe_status ag_expert(moe_ctx* c, int pass, void* X, cudaStream_t st) {
  const Dims& d = c->d;
  const size_t cnt = (size_t)d.Gep * d.Cs * d.H;
  NCCL_TRY(c, ncclGroupStart());
  for (int el = 0; el < d.El; ++el) {
    uint8_t* base = at<uint8_t>(X, (size_t)el * d.R * d.H * 2);
    NCCL_TRY(c, ncclAllGather(base + (size_t)d.t * cnt * 2, base, cnt, ncclBfloat16, c->comm->tp_comm, st));
  }
  NCCL_TRY(c, ncclGroupEnd());
  const int64_t xe = (int64_t)d.El * d.R * d.H * 2;
  ledger(c, MOE_COLL_ALLGATHER, pass, xe * (d.Gt - 1) / d.Gt);
  return MOE_OK;
}

// F8/B7 under DTD: in-place reduce-scatter of expert space over TP (AR + drop = RS).
moe_status rs_expert(moe_ctx* c, int pass, void* Y, cudaStream_t st, int el_lo = 0, int el_hi = -1,
                     bool count = true) {
  const Dims& d = c->d;
  const size_t cnt = (size_t)d.Gep * d.Cs * d.H;
  if (el_hi < 0) el_hi = d.El;
  NCCL_TRY(c, ncclGroupStart());
  for (int el = el_lo; el < el_hi; ++el) {
    uint8_t* base = at<uint8_t>(Y, (size_t)el * d.R * d.H * 2);
    NCCL_TRY(c, ncclReduceScatter(base, base + (size_t)d.t * cnt * 2, cnt, ncclBfloat16, ncclSum,
                                  c->comm->tp_comm, st));
  }
  NCCL_TRY(c, ncclGroupEnd());
  const int64_t xe = (int64_t)d.El * d.R * d.H * 2;
  if (count) ledger(c, MOE_COLL_REDUCESCATTER, pass, xe * (d.Gt - 1) / d.Gt);
  return MOE_OK;
}

// F8/B7 vanilla: the Megatron all-reduce of the row-parallel partials.
moe_status ar_expert(moe_ctx* c, int pass, void* Y, cudaStream_t st, int el_lo = 0, int el_hi = -1,
                     bool count = true) {
  const Dims& d = c->d;
  if (el_hi < 0) el_hi = d.El;
  const size_t per = (size_t)d.R * d.H;
  uint8_t* base = at<uint8_t>(Y, (size_t)el_lo * per * 2);
  NCCL_TRY(c, ncclAllReduce(base, base, per * (el_hi - el_lo), ncclBfloat16, ncclSum, c->comm->tp_comm, st));
  const size_t cnt = (size_t)d.El * per;
  if (count) ledger(c, MOE_COLL_ALLREDUCE, pass, 2 * (int64_t)cnt * 2 * (d.Gt - 1) / d.Gt);
  return MOE_OK;
}

// F10/B9: in-place all-gather of slot space over TP.
moe_status ag_slot(moe_ctx* c, int pass, void* O, cudaStream_t st) {
  const Dims& d = c->d;
  const size_t cnt = (size_t)d.E * d.Cs * d.H;
  NCCL_TRY(c, ncclAllGather(at<uint8_t>(O, (size_t)d.t * cnt * 2), O, cnt, ncclBfloat16, c->comm->tp_comm, st));
  ledger(c, MOE_COLL_ALLGATHER, pass, (int64_t)d.E * d.C * d.H * 2 * (d.Gt - 1) / d.Gt);
  return MOE_OK;
}

// cuStreamWaitValue32 through the runtime's driver entry point (no -lcuda); null if absent
using StreamWait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamWait32 stream_wait32() {
  static const StreamWait32 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return StreamWait32(nullptr);
    return reinterpret_cast<StreamWait32>(f);
  }();
  return fn;
}

moe_status gemm(moe_ctx* c, const GemmArgs& g, cudaStream_t st) {
  const char* why = "";
  if (c) {
    Scope sc_(c, MOE_K_GEMM, st, 1);
    cudaError_t e = gemm_tc(g, st, &why);
    if (e != cudaSuccess) {
      c->poisoned = true;
      return fail(MOE_ERR_CUDA, std::string("expert GEMM: ") + why + " (" + cudaGetErrorString(e) + ")");
    }
    return MOE_OK;
  }
  cudaError_t e = gemm_tc(g, st, &why);
  if (e != cudaSuccess) {
    if (c) c->poisoned = true;
    return fail(MOE_ERR_CUDA, std::string("expert GEMM: ") + why + " (" + cudaGetErrorString(e) + ")");
  }
  return MOE_OK;
}


// ---- peer-memory exchange (default for world > 1) ----
// Piece lists (static per config): "dispatch" moves slot-space pieces (D, dO) into
// expert-space windows (WX, WdY); "return" moves expert-space pieces (Ypart, dXp,
// after the TP reduction) into slot-space windows (WO, WdS). Under DTD a rank
// sends only its slot slice t, to every TP rank of the destination (the folded
// all-gather); vanilla sends all slices to the same-t rank only.
void build_pieces(const Dims& d, bool dispatch, std::vector<Piece>& v, int64_t bytes[3],
                  std::vector<int>* els = nullptr) {
  const uint64_t pb = (uint64_t)d.Cs * d.H * 2;
  const int lo = d.dtd ? d.t : 0, hi = d.dtd ? d.t + 1 : d.Gt;
  auto rank_of = [&](int ep, int t) { return (d.d * d.Gep + ep) * d.Gt + t; };
  auto push = [&](uint64_t so, uint64_t dof, int ep2, int t2) {
    Piece p;
    p.src_off = so;
    p.dst_off = dof;
    p.dst_rank = rank_of(ep2, t2);
    p.kind = (p.dst_rank == d.rank) ? 0 : (t2 == d.t ? 1 : 2);
    bytes[p.kind] += (int64_t)pb;
    v.push_back(p);
  };
  for (int i = 0; i < 3; ++i) bytes[i] = 0;
  if (dispatch) {
    for (int e = 0; e < d.E; ++e) {
      const int ep2 = e / d.El, el = e % d.El;
      for (int tt = lo; tt < hi; ++tt) {
        const uint64_t so = ((uint64_t)tt * d.E + e) * pb;
        const uint64_t dof = (((uint64_t)el * d.Gt + tt) * d.Gep + d.ep) * pb;
        if (d.dtd)
          for (int t2 = 0; t2 < d.Gt; ++t2) push(so, dof, ep2, t2);
        else
          push(so, dof, ep2, d.t);
      }
    }
  } else {
    for (int el = 0; el < d.El; ++el) {
      const int e = d.ep * d.El + el;
      for (int src = 0; src < d.Gep; ++src)
        for (int tt = lo; tt < hi; ++tt) {
          const uint64_t so = (((uint64_t)el * d.Gt + tt) * d.Gep + src) * pb;
          const uint64_t dof = ((uint64_t)tt * d.E + e) * pb;
          if (d.dtd)
            for (int t2 = 0; t2 < d.Gt; ++t2) push(so, dof, src, t2);
          else
            push(so, dof, src, d.t);
          if (els) els->resize(v.size(), el);
        }
    }
  }
}

// Per-layer exchange state over the communicator's windows: piece lists (the local
// return pieces live in the comm's device arena), the overlap stream and its events.
moe_status setup_peer(moe_ctx* c) {
  const Dims& d = c->d;
  moe_comm* m = c->comm;
  std::vector<Piece> disp, ret;
  build_pieces(d, true, disp, c->disp_bytes);
  build_pieces(d, false, ret, c->ret_bytes, &c->h_ret_el);
  c->h_ret = ret;
  std::vector<Piece> loc;
  for (const Piece& p : ret)
    if (p.dst_rank == d.rank) loc.push_back(p);
  c->n_ret_local = (int)loc.size();
  c->d_ret_local = comm_pieces(m, (int)loc.size());
  if (!c->d_ret_local) return fail(MOE_ERR_STATE, "communicator piece arena exhausted (too many layers)");
  if (!loc.empty())
    CUDA_TRY(c, cudaMemcpy(c->d_ret_local, loc.data(), sizeof(Piece) * loc.size(), cudaMemcpyHostToDevice));
  c->gsig = reinterpret_cast<int32_t*>(comm_pieces(m, (8 * sizeof(int32_t) + sizeof(Piece) - 1) / sizeof(Piece)));
  if (!c->gsig) return fail(MOE_ERR_STATE, "communicator piece arena exhausted (too many layers)");
  CUDA_TRY(c, cudaMemset(c->gsig, 0, 8 * sizeof(int32_t)));
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  for (int i = 0; i < 4; ++i) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  for (int i = 0; i < 4; ++i) CUDA_TRY(c, cudaEventCreateWithFlags(&c->evp[i], cudaEventDisableTiming));
  return MOE_OK;
}

void teardown_peer(moe_ctx* c) {
  if (c->side) cudaStreamDestroy(c->side);
  c->side = nullptr;
  for (int i = 0; i < 4; ++i) {
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->evp[i]) cudaEventDestroy(c->evp[i]);
    c->ev[i] = c->evp[i] = nullptr;
  }
}

PeerDst peer_dst(const moe_ctx* c, int win) {
  const Dims& d = c->d;
  PeerDst pd;
  pd.table = c->comm->d_table;
  pd.nwin = c->comm->nwin;
  pd.win = win;
  pd.d = d.d; pd.ep = d.ep; pd.t = d.t; pd.Gt = d.Gt; pd.Gep = d.Gep; pd.El = d.El;
  // folded all-gather: write every TP rank of the destination (DTD, and NVLS direct where the
  // own group's rows take one multicast store); two-step NVLS sends the own slice to the same t
  pd.dtd = d.dtd && (!d.nvls || d.nvls_direct) ? 1 : 0;
  pd.mc = d.nvls_direct && !c->comm->mcwin.empty() ? c->comm->mcwin[win] : nullptr;
  return pd;
}

// A deadline failure of the communicator (device-side spin or emulated host barrier)
// poisons the context and is reported as MOE_ERR_TIMEOUT.
moe_status check_comm(moe_ctx* c) {
  std::string why;
  const moe_status s = comm_check(c->comm, &why);
  if (s != MOE_OK) {
    c->poisoned = true;
    return fail(s, why);
  }
  return MOE_OK;
}

#define TRY0(expr)                        \
  do {                                    \
    moe_status _s0 = (expr);              \
    if (_s0 != MOE_OK) return _s0;        \
  } while (0)

// Return-direction exchange of the remote pieces on the copy engines (no SMs): one peer
// cudaMemcpyAsync per piece of local experts [el_lo, el_hi), so it overlaps a persistent
// GEMM. This rank's own pieces go through exchange_local (an SM copy kernel), since a
// same-device memcpy would itself wait for free SMs.
moe_status exchange_ce(moe_ctx* c, const void* src, int win, int el_lo, int el_hi, cudaStream_t st) {
  const Dims& d = c->d;
  const size_t pb = (size_t)d.Cs * d.H * 2;
  for (size_t i = 0; i < c->h_ret.size(); ++i) {
    const int el = c->h_ret_el[i];
    if (el < el_lo || el >= el_hi) continue;
    const Piece& p = c->h_ret[i];
    if (p.dst_rank == d.rank) continue;
    uint8_t* dst = static_cast<uint8_t*>(c->comm->h_table[(size_t)p.dst_rank * c->comm->nwin + win]) + p.dst_off;
    CUDA_TRY(c, cudaMemcpyAsync(dst, static_cast<const uint8_t*>(src) + p.src_off, pb,
                                cudaMemcpyDeviceToDevice, st));
  }
  return MOE_OK;
}

// Dispatch-direction pieces of the G_t = 1 split exchange on the copy engines: the staged
// slot-space rows of every remote rank's experts go into that rank's window at source
// block `me` ([E_l][G_ep][C][H]).
// Per-source pipelined variant: the pieces for each destination (staggered order
// me+1, me+2, ... so that every rank receives from one source at a time) followed by a
// readiness flag in that destination's flag region; returns the epoch to wait for.
moe_status exchange_ce_dispatch_sig(moe_ctx* c, const void* stage, int win, cudaStream_t st, uint32_t* epoch) {
  const Dims& d = c->d;
  moe_comm* m = c->comm;
  const size_t pb = (size_t)d.C * d.H * 2;
  const uint32_t ep = ++m->sig_epoch;
  *epoch = ep;
  for (int k = 1; k < d.Gep; ++k) {
    const int ep2 = (d.ep + k) % d.Gep;
    const int r = d.d * d.Gep + ep2;  // G_t = 1
    for (int el = 0; el < d.El; ++el) {
      const uint8_t* src = static_cast<const uint8_t*>(stage) + (size_t)(ep2 * d.El + el) * pb;
      uint8_t* dst = static_cast<uint8_t*>(m->h_table[(size_t)r * m->nwin + win]) +
                     ((size_t)el * d.Gep + d.ep) * pb;
      CUDA_TRY(c, cudaMemcpyAsync(dst, src, pb, cudaMemcpyDeviceToDevice, st));
    }
    std::string why;
    const moe_status s = comm_signal(m, r, ep, st, &why);
    if (s != MOE_OK) { c->poisoned = true; return fail(s, why); }
    if (m->tr == TR_IPC) c->stats.kernel_launches[MOE_K_COMM] += 1;
  }
  return MOE_OK;
}

// Waits (on st) until source block `src`'s pieces of exchange `epoch` are in this rank's window.
moe_status wait_source(moe_ctx* c, int src, uint32_t epoch, cudaStream_t st) {
  moe_comm* m = c->comm;
  std::string why;
  const moe_status s = comm_wait(m, c->d.d * c->d.Gep + src, epoch, st, &why);  // G_t = 1: rank = d*G_ep + ep
  if (s != MOE_OK) { c->poisoned = true; return fail(s, why); }
  if (m->tr == TR_IPC) c->stats.kernel_launches[MOE_K_COMM] += 1;
  return MOE_OK;
}

// Expert GEMM over the rows of source blocks [s0, s1) of every local expert (rows
// [s0*C, s1*C) of each [G_ep*C]-row batch): strided batches, G_t = 1 split exchange.
moe_status gemm_rows(moe_ctx* c, GemmArgs g, int s0, int s1, int64_t a_ld, int64_t d_ld, cudaStream_t st) {
  const Dims& d = c->d;
  if (s1 <= s0) return MOE_OK;
  const int64_t r0 = (int64_t)s0 * d.C;
  g.M = (int)((s1 - s0) * d.C);
  g.A = static_cast<const uint8_t*>(g.A) + (size_t)r0 * a_ld * 2;
  g.D = static_cast<uint8_t*>(g.D) + (size_t)r0 * d_ld * 2;
  if (g.aux) g.aux = static_cast<uint8_t*>(g.aux) + (size_t)r0 * d_ld * 2;
  g.a_bs = d.R * a_ld;
  g.d_bs = d.R * d_ld;
  return gemm(c, g, st);
}

// G_t = 1 split exchange, GEMM1 / B4: the own source block, then the remote blocks in
// arrival order (me-1, me-2, ...) in groups of g, each group one launch after its pieces
// are in. g = 1 unless one block is too few tiles for the persistent grid (EP8: 2 local
// experts x 4 x 32 = 256 tiles = 3.5 waves of 74 CTA pairs, ~13 % tail): then g blocks
// per launch bring it to >= ~6 waves; blocks still arrive faster than they are consumed.
moe_status gemm_sources(moe_ctx* c, const GemmArgs& g, uint32_t sig, int64_t a_ld, int64_t d_ld, cudaStream_t st) {
  const Dims& d = c->d;
  TRY0(gemm_rows(c, g, d.ep, d.ep + 1, a_ld, d_ld, st));  // own block overlaps the copy engines
  const int64_t tiles = (int64_t)d.El * ((d.C + 255) / 256) * ((g.N + 255) / 256);
  const int64_t want = 6 * 74;
  int grp = tiles > 0 ? (int)((want + tiles - 1) / tiles) : 1;
  if (grp < 1) grp = 1;
  for (int k0 = 1; k0 < d.Gep; k0 += grp) {
    const int k1 = k0 + grp < d.Gep ? k0 + grp : d.Gep;
    {
      Scope sc_(c, MOE_K_COMM, st, 0);
      for (int k = k0; k < k1; ++k) TRY0(wait_source(c, (d.ep - k + d.Gep) % d.Gep, sig, st));
    }
    // sources me-k1+1 .. me-k0 (mod G_ep): contiguous unless they wrap past 0
    const int lo = d.ep - (k1 - 1), hi = d.ep - k0 + 1;  // [lo, hi) before the wrap
    if (lo >= 0) {
      TRY0(gemm_rows(c, g, lo, hi, a_ld, d_ld, st));
    } else {
      if (hi > 0) TRY0(gemm_rows(c, g, 0, hi, a_ld, d_ld, st));
      TRY0(gemm_rows(c, g, lo + d.Gep, hi > 0 ? d.Gep : hi + d.Gep, a_ld, d_ld, st));
    }
  }
  return MOE_OK;
}

// G_t > 1: barrier (every TP partial complete), fused TP reduction + return exchange,
// barrier (every destination written). Same ledger as the NCCL-mode RS/AR + a2a (+AG).
moe_status tp_return(moe_ctx* c, int pass, int src_win, int dst_win, cudaStream_t st);

moe_status exchange_local(moe_ctx* c, const void* src, int win, cudaStream_t st) {
  const Dims& d = c->d;
  CUDA_TRY(c, peer_exchange(src, c->comm->d_table, c->comm->nwin, win, c->d_ret_local, c->n_ret_local,
                            (size_t)d.Cs * d.H * 2, st));
  c->stats.kernel_launches[MOE_K_COMM] += 1;
  return MOE_OK;
}

moe_status barrier(moe_ctx* c, cudaStream_t st) {
  std::string why;
  const moe_status s = comm_barrier(c->comm, st, &why);
  if (s != MOE_OK) { c->poisoned = true; return fail(s, why); }
  if (c->comm->tr == TR_IPC) c->stats.kernel_launches[MOE_K_COMM] += 1;
  return MOE_OK;
}

// All-gather egress of a folded exchange: the G_t - 1 copies a rank writes itself, or under
// NVLS direct (every destination is the own TP group) the one copy that goes through the
// multicast mapping.
int64_t ag_bytes(const Dims& d, int64_t folded) { return d.nvls_direct ? folded / (d.Gt - 1) : folded; }

// MOE_F_NVLS: DTD's all-gather as its own step — this rank's slice of window `win`
// (expert space [E_l][G_t][G_ep][C_s][H] or slot space [G_t][E][C_s][H]) goes once through
// the TP group's multicast mapping (emulated ranks: a store per TP peer), then a barrier.
moe_status nvls_allgather(moe_ctx* c, int win, bool expert_space, int pass, cudaStream_t st) {
  const Dims& d = c->d;
  moe_comm* m = c->comm;
  TpAllGather ag;
  ag.table = m->d_table;
  ag.nwin = m->nwin;
  ag.win = win;
  ag.rank = d.rank;
  ag.tp0 = d.rank - d.t;
  ag.Gt = d.Gt;
  ag.mc = m->mcwin.empty() ? nullptr : m->mcwin[win];
  const uint64_t row = (uint64_t)d.H * 2;
  if (expert_space) {
    ag.seg_bytes = (uint64_t)d.Gep * d.Cs * row;
    ag.stride = (uint64_t)d.Gt * ag.seg_bytes;
    ag.nseg = d.El;
  } else {
    ag.seg_bytes = (uint64_t)d.E * d.Cs * row;
    ag.stride = 0;
    ag.nseg = 1;
  }
  ag.base_off = (uint64_t)d.t * ag.seg_bytes;
  CUDA_TRY(c, tp_allgather(ag, st));  // timed inside the caller's comm scope
  c->stats.kernel_launches[MOE_K_COMM] += 1;
  TRY0(barrier(c, st));
  ledger(c, MOE_COLL_ALLGATHER, pass, (int64_t)(ag.seg_bytes * ag.nseg));  // egress: the slice, once
  return MOE_OK;
}

moe_status tp_return(moe_ctx* c, int pass, int src_win, int dst_win, cudaStream_t st) {
  const Dims& d = c->d;
  TRY0(barrier(c, st));
  ReduceReturn rr;
  rr.table = c->comm->d_table;
  rr.nwin = c->comm->nwin;
  rr.src_win = src_win;
  rr.dst_win = dst_win;
  rr.d = d.d; rr.ep = d.ep; rr.t = d.t; rr.Gt = d.Gt; rr.Gep = d.Gep; rr.El = d.El; rr.E = d.E; rr.H = d.H;
  rr.Cs = d.Cs;
  rr.dtd = d.dtd ? 1 : 0;
  rr.fold = d.dtd && (!d.nvls || d.nvls_direct) ? 1 : 0;
  rr.mc = d.nvls_direct && !c->comm->mcwin.empty() ? c->comm->mcwin[dst_win] : nullptr;
  CUDA_TRY(c, reduce_return(rr, st));
  c->stats.kernel_launches[MOE_K_COMM] += 1;
  TRY0(barrier(c, st));
  const int64_t xe = (int64_t)d.El * d.R * d.H * 2;
  if (d.dtd) ledger(c, MOE_COLL_REDUCESCATTER, pass, xe * (d.Gt - 1) / d.Gt);
  else ledger(c, MOE_COLL_ALLREDUCE, pass, 2 * xe * (d.Gt - 1) / d.Gt);
  if (d.Gep > 1) ledger(c, MOE_COLL_A2A, pass, c->ret_bytes[1]);
  if (d.nvls && !d.nvls_direct) TRY0(nvls_allgather(c, dst_win, false, pass, st));
  else if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, pass, ag_bytes(d, c->ret_bytes[2]));
  return MOE_OK;
}

// Barrier publishing a fused peer write (dispatch / combine-backward) + ledger.
moe_status publish(moe_ctx* c, bool dispatch, int pass, cudaStream_t st) {
  const Dims& d = c->d;
  TRY0(barrier(c, st));
  const int64_t* b = dispatch ? c->disp_bytes : c->ret_bytes;
  if (d.Gep > 1) ledger(c, MOE_COLL_A2A, pass, b[1]);
  if (d.dtd && (!d.nvls || d.nvls_direct)) ledger(c, MOE_COLL_ALLGATHER, pass, ag_bytes(d, b[2]));
  return MOE_OK;
}

#define TRY(expr)                         \
  do {                                    \
    moe_status _s = (expr);               \
    if (_s != MOE_OK) return _s;          \
  } while (0)

}  // namespace

// F3-F11 of one forward on an already-routed saved blob. pass 0: the forward
// (y written); pass 2: a plain-checkpointing replay (y == nullptr, every collective
// re-issued and counted as replay). rslot: ring slot of the peer windows.
moe_status forward_core(moe_ctx* c, const void* x, const void* w1, const void* w2, void* y,
                        void* saved, cudaStream_t st, int pass, int rslot) {
  const Dims& d = c->d;
  const SavedLayout& sv = c->sv;
  const ScratchLayout& sc = c->sc;
  const SlotSpace ss = slot_space(d);
  const bool solo = d.world == 1;
  const int lo = d.dtd ? d.t : 0, hi = d.dtd ? d.t + 1 : d.Gt;
  // F3 dispatch (DTD: only this rank's slot slice), F4 a2a, F5 all-gather
  void* X = d.peer ? c->comm->win[c->comm->wx(rslot)] : at<uint8_t>(saved, sv.X);
  const int32_t* tok_of = at<int32_t>(saved, sv.tok_of);
  const int32_t* count = at<int32_t>(saved, sv.count);
  void* D = sc.D_in_saved ? X : at<uint8_t>(c->scratch, sc.D);
  // G_t = 1 split exchange: local rows -> own window, remote rows -> stage -> copy engines,
  // overlapped with GEMM1 on the local source block
  const bool split = d.peer && d.Gt == 1 && d.Gep > 1 && c->overlap;
  uint32_t sig = 0;
  // One GPU, top-1: F11 fused into F7's epilogue (O still stored for the backward); the
  // dispatch launch zeroes the y rows of dropped tokens
  const bool fused_combine = solo && d.K == 1 && y && !c->no_fused_combine;
  if (split) {
    SplitDst sd{X, D, d.ep, d.El, d.Gep};
    {
      Scope sc_(c, MOE_K_DISPATCH, st, 1);
      CUDA_TRY(c, dispatch_split(x, tok_of, count, ss, sd, st));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[3], st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[3], 0));
    {
      Scope sx_(c, MOE_K_XFER, c->side, 0);
      TRY(exchange_ce_dispatch_sig(c, D, c->comm->wx(rslot), c->side, &sig));
    }
    ledger(c, MOE_COLL_A2A, pass, c->disp_bytes[1]);
  } else if (d.peer) {
    // fused: rows go straight from x into the peers' expert-space windows
    {
      Scope sc_(c, MOE_K_DISPATCH, st, 1);
      CUDA_TRY(c, dispatch_peer(x, tok_of, count, ss, lo, hi, peer_dst(c, c->comm->wx(rslot)), st));
    }
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(publish(c, true, pass, st));
    if (d.nvls && !d.nvls_direct) TRY(nvls_allgather(c, c->comm->wx(rslot), true, pass, st));
  } else {
    Scope sc_(c, MOE_K_DISPATCH, st, 1);
    CUDA_TRY(c, dispatch(x, tok_of, count, ss, lo, hi, D, at<int32_t>(saved, sv.slot), d.T,
                         fused_combine ? y : nullptr, st));
  }
  if (!solo && !d.peer) {
    Scope sc_(c, MOE_K_COMM, st, 0);
    {
      TRY(ep_exchange(c, 0, pass, D, X, lo, hi, st));
      if (d.dtd) TRY(ag_expert(c, pass, X, st));
    }
  }
  if (d.peer && d.ckpt && !split) {  // CAC stash of the first collective's output
    Scope sc_(c, MOE_K_COMM, st, 0);
    CUDA_TRY(c, cudaMemcpyAsync(at<uint8_t>(saved, sv.X), X, (size_t)d.El * d.R * d.H * 2,
                                cudaMemcpyDeviceToDevice, st));
  }

  // F6 GEMM1 + GeLU (stores A = gelu(Hpre) and G = gelu'(Hpre)), F7 GEMM2
  void* G = d.ckpt ? at<uint8_t>(c->scratch, sc.Grec) : at<uint8_t>(saved, sv.G);
  void* A = d.ckpt ? at<uint8_t>(c->scratch, sc.Arec) : at<uint8_t>(saved, sv.A);
  void* O = d.peer ? c->comm->win[c->comm->wo(rslot)] : at<uint8_t>(saved, sv.O);
  void* Y = sc.Y_in_saved ? O : (d.peer && d.Gt > 1 ? c->comm->win[moe_comm::W_Y] : at<uint8_t>(c->scratch, sc.Ypart));
  GemmArgs g1{d.El, (int)d.R, d.Fl, d.H, X, 0, w1, 0, G, EPI_GELU, A};
  if (split) {
    // own block first (already in place), then each source block as its pieces land
    // (source me-k sends to me as its k-th destination)
    TRY(gemm_sources(c, g1, sig, d.H, d.Fl, st));
    if (d.ckpt) {  // CAC stash of the first collective's output
      Scope sc_(c, MOE_K_COMM, st, 0);
      CUDA_TRY(c, cudaMemcpyAsync(at<uint8_t>(saved, sv.X), X, (size_t)d.El * d.R * d.H * 2,
                                  cudaMemcpyDeviceToDevice, st));
    }
  } else {
    TRY(gemm(c, g1, st));
  }
  if (d.peer && d.Gt > 1) {
    // F7 GEMM2 into the TP-visible window, then F8-F10 as one fused kernel over peer
    // memory (NCCL's reduce-scatter would wait for the persistent GEMMs to free SMs)
    GemmArgs g2{d.El, (int)d.R, d.H, d.Fl, A, 0, w2, 0, Y, EPI_STORE, nullptr};
    TRY(gemm(c, g2, st));
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(tp_return(c, pass, moe_comm::W_Y, c->comm->wo(rslot), st));
    if (d.ckpt) {  // CAC stash of the second collective's output
      CUDA_TRY(c, cudaMemcpyAsync(at<uint8_t>(saved, sv.O), O, (size_t)d.E * d.C * d.H * 2,
                                  cudaMemcpyDeviceToDevice, st));
    }
  } else if (d.peer && split && !c->no_fused_return) {
    // (G_t = 1, split exchange) F7 + F9 fused: GEMM2's epilogue stores every row straight
    // into the slot-space window of its source rank over peer memory (the own rows into the
    // own window), so the return all-to-all overlaps the math tile by tile and needs no
    // copy engines, part launches or staging; one barrier publishes the windows.
    GemmArgs g2{d.El, (int)d.R, d.H, d.Fl, A, 0, w2, 0, Y, EPI_STORE, nullptr};
    PeerOut po;
    po.table = c->comm->d_table;
    po.nwin = c->comm->nwin;
    po.win = c->comm->wo(rslot);
    po.rank0 = d.d * d.Gep;  // G_t = 1: rank = d * G_ep + ep
    po.e0 = d.ep * d.El;
    po.C = d.C;
    g2.po = &po;
    TRY(gemm(c, g2, st));
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(barrier(c, st));
    if (d.Gep > 1) ledger(c, MOE_COLL_A2A, pass, c->ret_bytes[1]);
    if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, pass, c->ret_bytes[2]);
    if (d.ckpt) {  // CAC stash of the second collective's output
      CUDA_TRY(c, cudaMemcpyAsync(at<uint8_t>(saved, sv.O), O, (size_t)d.E * d.C * d.H * 2,
                                  cudaMemcpyDeviceToDevice, st));
    }
  } else if (d.peer) {
    // (G_t = 1) F7 GEMM2 in up to 4 expert parts; each part's return pieces (F9) go out on
    // the side stream (copy engines) while the next part computes, so only the last part's
    // pieces are exposed
    const int P = c->overlap ? (d.El < 4 ? d.El : 4) : 1;
    const size_t rows = (size_t)d.R * d.H;
    if (P > 1 && stream_wait32() && !c->no_gemm_signal) {
      // one GEMM2 launch (no per-part tail waves); each part's last tile raises its flag
      // and the side stream's copy engines start that part's return pieces (F9)
      GemmSignal gs;
      gs.cnt = c->gsig;
      gs.flag = reinterpret_cast<uint32_t*>(c->gsig + 4);
      gs.epoch = ++c->gsig_epoch;
      gs.nparts = P;
      for (int q = 0; q <= P; ++q) gs.part_b[q] = q * d.El / P;
      GemmArgs g2{d.El, (int)d.R, d.H, d.Fl, A, 0, w2, 0, Y, EPI_STORE, nullptr};
      g2.sig = &gs;
      TRY(gemm(c, g2, st));
      // the waits go in after the GEMM launch: a stream-ordered value wait may block a
      // hardware queue shared with other streams, so the work it waits for must already
      // be enqueued (same rule as an event wait)
      for (int q = 0; q < P; ++q) {
        if (gs.part_b[q + 1] <= gs.part_b[q]) continue;
        const CUresult r = stream_wait32()(c->side, reinterpret_cast<CUdeviceptr>(gs.flag + q), gs.epoch,
                                           CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) {
          c->poisoned = true;
          return fail(MOE_ERR_CUDA, "cuStreamWaitValue32 failed");
        }
        Scope sx_(c, MOE_K_XFER, c->side, 0);
        TRY(exchange_ce(c, Y, c->comm->wo(rslot), gs.part_b[q], gs.part_b[q + 1], c->side));
      }
    } else
    for (int part = 0; part < P; ++part) {
      const int e0 = part * d.El / P, e1 = (part + 1) * d.El / P;
      if (e1 <= e0) continue;
      const size_t ao = (size_t)e0 * d.R * d.Fl * 2, yo = (size_t)e0 * rows * 2;
      GemmArgs g2{e1 - e0, (int)d.R, d.H, d.Fl, at<uint8_t>(A, ao), 0,
                  at<uint8_t>(const_cast<void*>(w2), (size_t)e0 * d.H * d.Fl * 2), 0,
                  at<uint8_t>(Y, yo), EPI_STORE, nullptr};
      TRY(gemm(c, g2, st));
      CUDA_TRY(c, cudaEventRecord(c->evp[part], st));
      CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->evp[part], 0));
      {
        Scope sx_(c, MOE_K_XFER, c->side, 0);
        TRY(exchange_ce(c, Y, c->comm->wo(rslot), e0, e1, c->side));
      }
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[2], c->side));
    Scope sc_(c, MOE_K_COMM, st, 0);
    // the own pieces (SM copy) need only GEMM2's output: they overlap the side stream's
    // last copy-engine pieces instead of following them
    TRY(exchange_local(c, Y, c->comm->wo(rslot), st));
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev[2], 0));
    TRY(barrier(c, st));
    if (d.Gep > 1) ledger(c, MOE_COLL_A2A, pass, c->ret_bytes[1]);
    if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, pass, c->ret_bytes[2]);
    if (d.ckpt) {  // CAC stash of the second collective's output
      CUDA_TRY(c, cudaMemcpyAsync(at<uint8_t>(saved, sv.O), O, (size_t)d.E * d.C * d.H * 2,
                                  cudaMemcpyDeviceToDevice, st));
    }
  } else {
    GemmArgs g2{d.El, (int)d.R, d.H, d.Fl, A, 0, w2, 0, Y, EPI_STORE, nullptr};
    GateDxArgs cmb{at<int32_t>(saved, sv.tok_of), at<int32_t>(saved, sv.count), nullptr, nullptr, d.E, d.C, y,
                   at<float>(saved, sv.prob), nullptr, nullptr};
    if (fused_combine) {
      g2.epilogue = EPI_COMBINE;
      g2.gdx = &cmb;
    }
    TRY(gemm(c, g2, st));
    // F8 TP reduce, F9 a2a back, F10 all-gather
    if (!solo) {
      Scope sc_(c, MOE_K_COMM, st, 0);
      if (d.Gt > 1) {
        if (d.dtd) TRY(rs_expert(c, pass, Y, st));
        else TRY(ar_expert(c, pass, Y, st));
      }
      TRY(ep_exchange(c, 1, pass, O, Y, lo, hi, st));
      if (d.dtd) TRY(ag_slot(c, pass, O, st));
    }
  }

  // F11 combine (not in a checkpoint replay: the layer output is not needed again)
  if (y && !fused_combine) {
    Scope sc_(c, MOE_K_COMBINE, st, 1);
    CUDA_TRY(c, combine(O, at<int32_t>(saved, sv.expert), at<int32_t>(saved, sv.slot),
                        at<float>(saved, sv.prob), ss, d.T, y, st));
  }
  return MOE_OK;
}

extern "C" {

const char* moe_status_string(moe_status s) {
  switch (s) {
    case MOE_OK: return "MOE_OK";
    case MOE_ERR_ARG: return "MOE_ERR_ARG";
    case MOE_ERR_SHAPE: return "MOE_ERR_SHAPE";
    case MOE_ERR_ALIGN: return "MOE_ERR_ALIGN";
    case MOE_ERR_STATE: return "MOE_ERR_STATE";
    case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
    case MOE_ERR_NCCL: return "MOE_ERR_NCCL";
    case MOE_ERR_UNSUPPORTED: return "MOE_ERR_UNSUPPORTED";
    case MOE_ERR_TIMEOUT: return "MOE_ERR_TIMEOUT";
  }
  return "MOE_ERR_UNKNOWN";
}

const char* moe_last_error_detail(void) { return g_detail.c_str(); }

moe_status moe_plan_layout(const moe_config* cfg, int world, int rank, moe_layout* out) {
  if (!out) return fail(MOE_ERR_ARG, "null output");
  Dims d;
  std::string why;
  moe_status s = make_dims(cfg, world, rank, &d, &why);
  if (s != MOE_OK) return fail(s, why);
  out->world = world; out->rank = rank;
  out->d = d.d; out->ep = d.ep; out->t = d.t;
  out->experts_local = d.El; out->ffn_local = d.Fl;
  out->capacity = d.C; out->slot_slice = d.Cs; out->rows_per_expert = d.R;
  out->token_groups = d.S;
  return MOE_OK;
}

moe_status moe_plan_bytes(const moe_config* cfg, int world, int rank, size_t* saved_bytes,
                          size_t* scratch_bytes) {
  Dims d;
  std::string why;
  moe_status s = make_dims(cfg, world, rank, &d, &why);
  if (s != MOE_OK) return fail(s, why);
  SavedLayout sv;
  ScratchLayout sc;
  make_layouts(d, &sv, &sc);
  if (saved_bytes) *saved_bytes = sv.total;
  if (scratch_bytes) *scratch_bytes = sc.total;
  return MOE_OK;
}

moe_status moe_plan_collectives(const moe_config* cfg, int world, int rank, moe_collective* out,
                                int cap, int* n) {
  if (!n) return fail(MOE_ERR_ARG, "null count");
  Dims d;
  std::string why;
  moe_status s = make_dims(cfg, world, rank, &d, &why);
  if (s != MOE_OK) return fail(s, why);
  std::vector<moe_collective> v = make_schedule(d);
  *n = (int)v.size();
  if (out && cap >= (int)v.size()) std::memcpy(out, v.data(), v.size() * sizeof(moe_collective));
  return MOE_OK;
}

moe_status moe_get_unique_id(uint8_t uid[128]) {
  if (!uid) return fail(MOE_ERR_ARG, "null uid");
  ncclUniqueId id;
  NCCL_TRY((moe_ctx*)nullptr, ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(uid, &id, 128);
  return MOE_OK;
}

}  // extern "C"

namespace {

// A layer context on communicator m (nullptr when world == 1).
moe_status make_ctx(const moe_config* cfg, moe_comm* m, int world, int rank, void* scratch,
                    size_t scratch_bytes, moe_ctx** out) {
  Dims d;
  std::string why;
  moe_status s = make_dims(cfg, world, rank, &d, &why);
  if (s != MOE_OK) return fail(s, why);
  moe_ctx* c = new moe_ctx();
  {
    const char* nf = std::getenv("MOE_NO_FUSED_DX");
    c->no_fused_dx = nf && nf[0] == '1';
    const char* nc = std::getenv("MOE_NO_FUSED_COMBINE");
    c->no_fused_combine = nc && nc[0] == '1';
    const char* no = std::getenv("MOE_NO_OVERLAP");
    c->overlap = !(no && no[0] == '1');
    const char* ns = std::getenv("MOE_NO_GEMM_SIGNAL");
    c->no_gemm_signal = ns && ns[0] == '1';
    const char* nr = std::getenv("MOE_NO_FUSED_RETURN");
    c->no_fused_return = nr && nr[0] == '1';
  }
  c->d = d;
  c->cfg = *cfg;
  c->timing = (cfg->flags & MOE_F_TIMING) != 0;
  make_layouts(d, &c->sv, &c->sc);
  std::memset(&c->stats, 0, sizeof(c->stats));
  if (!scratch || scratch_bytes < c->sc.total) {
    delete c;
    return fail(MOE_ERR_ARG, "scratch missing or smaller than moe_plan_bytes");
  }
  if (reinterpret_cast<uintptr_t>(scratch) & 255) {
    delete c;
    return fail(MOE_ERR_ALIGN, "scratch must be 256-byte aligned");
  }
  c->scratch = static_cast<uint8_t*>(scratch);
  c->scratch_bytes = scratch_bytes;
  if (world > 1) {
    // the layer must fit the communicator it is attached to
    CommPlan need;
    s = make_comm_plan(cfg, 1, world, rank, &need, &why);
    const CommPlan& have = m->plan;
    if (s == MOE_OK) {
      if (have.world != world || have.rank != rank || have.Gt != d.Gt || have.Gep != d.Gep) {
        s = MOE_ERR_ARG;
        why = "layer's world/rank/g_tensor/g_expert differ from the communicator's";
      } else if (need.peer && (!have.peer || need.expert_space > have.expert_space ||
                               need.slot_space > have.slot_space || need.tp_space > have.tp_space)) {
        s = MOE_ERR_ARG;
        why = "layer needs larger peer windows than the communicator was planned for";
      } else if (need.nccl && !m->tp_comm) {
        s = MOE_ERR_STATE;
        why = "MOE_F_NCCL_EXCHANGE layer on a communicator planned without it";
      }
    }
    if (s != MOE_OK) { delete c; return fail(s, why); }
    c->comm = m;
    if (d.peer) {
      s = setup_peer(c);
      if (s != MOE_OK) {
        const std::string why2 = g_detail;
        teardown_peer(c);
        delete c;
        return fail(s, "peer-memory exchange setup: " + why2);
      }
    }
    m->refs += 1;
  }
  *out = c;
  return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_comm_plan_bytes(const moe_config* cfgs, int n, int world, int rank, size_t* device_bytes) {
  if (!device_bytes) return fail(MOE_ERR_ARG, "null output");
  CommPlan p;
  std::string why;
  moe_status s = make_comm_plan(cfgs, n, world, rank, &p, &why);
  if (s != MOE_OK) return fail(s, why);
  *device_bytes = p.total;
  return MOE_OK;
}

moe_status moe_comm_create(const moe_config* cfgs, int n, const uint8_t uid[128], int world, int rank,
                           moe_comm** out) {
  if (!out) return fail(MOE_ERR_ARG, "null comm output");
  if (world < 2) return fail(MOE_ERR_ARG, "a communicator needs world > 1");
  std::string why;
  moe_status s = comm_create(cfgs, n, uid, nullptr, world, rank, out, &why);
  if (s != MOE_OK) return fail(s, why);
  return MOE_OK;
}

moe_status moe_comm_create_emulated(const moe_config* cfgs, int n, moe_emu_group* group, int rank,
                                    moe_comm** out) {
  if (!out || !group) return fail(MOE_ERR_ARG, "null group / comm output");
  int world = 0;
  world = emu_world(group);
  moe_status s;
  if (world < 2) return fail(MOE_ERR_ARG, "an emulated group needs world > 1");
  std::string why;
  s = comm_create(cfgs, n, nullptr, group, world, rank, out, &why);
  if (s != MOE_OK) return fail(s, why);
  return MOE_OK;
}

moe_status moe_comm_destroy(moe_comm* m) {
  if (!m) return MOE_OK;
  if (m->refs > 0) return fail(MOE_ERR_STATE, "layer contexts still attached to the communicator");
  cudaDeviceSynchronize();
  comm_destroy(m);
  return MOE_OK;
}

moe_status moe_create(const moe_config* cfg, const uint8_t uid[128], int world, int rank,
                      void* scratch, size_t scratch_bytes, moe_ctx** out) {
  if (!out) return fail(MOE_ERR_ARG, "null ctx output");
  *out = nullptr;
  Dims d;
  std::string why;
  moe_status s = make_dims(cfg, world, rank, &d, &why);
  if (s != MOE_OK) return fail(s, why);
  moe_comm* m = nullptr;
  if (world > 1) {
    if (!uid) return fail(MOE_ERR_ARG, "uid required when world > 1");
    s = comm_create(cfg, 1, uid, nullptr, world, rank, &m, &why);
    if (s != MOE_OK) return fail(s, why);
    m->private_to_ctx = true;
  }
  s = make_ctx(cfg, m, world, rank, scratch, scratch_bytes, out);
  if (s != MOE_OK && m) {
    const std::string keep = g_detail;
    comm_destroy(m);
    g_detail = keep;
  }
  return s;
}

moe_status moe_create_on_comm(const moe_config* cfg, moe_comm* comm, void* scratch, size_t scratch_bytes,
                              moe_ctx** out) {
  if (!out || !comm) return fail(MOE_ERR_ARG, "null comm / ctx output");
  *out = nullptr;
  return make_ctx(cfg, comm, comm->plan.world, comm->plan.rank, scratch, scratch_bytes, out);
}

moe_status moe_destroy(moe_ctx* c) {
  if (!c) return MOE_OK;
  moe_comm* m = c->comm;
  if (m) {
    cudaDeviceSynchronize();
    teardown_peer(c);
    m->refs -= 1;
    if (m->private_to_ctx) comm_destroy(m);
  }
  delete c;
  return MOE_OK;
}

moe_status moe_forward(moe_ctx* c, const void* x, const float* wg, const void* w1, const void* w2,
                       void* y, void* saved, const int32_t* forced_expert, void* stream) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (c->poisoned) return fail(MOE_ERR_STATE, "ctx poisoned by an earlier CUDA/NCCL failure");
  if (c->comm) TRY(check_comm(c));
  if (!x || !wg || !w1 || !w2 || !y || !saved) return fail(MOE_ERR_ARG, "null tensor pointer");
  if (c->d.forced != (forced_expert != nullptr))
    return fail(MOE_ERR_ARG, "forced_expert must be given iff MOE_F_FORCED_ROUTING");
  if (!aligned16(x) || !aligned16(wg) || !aligned16(w1) || !aligned16(w2) || !aligned16(y))
    return fail(MOE_ERR_ALIGN, "tensor pointers must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(saved) & 255) return fail(MOE_ERR_ALIGN, "saved must be 256-byte aligned");
  const Dims& d = c->d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const SavedLayout& sv = c->sv;
  const ScratchLayout& sc = c->sc;

  // F1 + F2: gate and capacity slots
  RouteArgs ra;
  ra.x = x; ra.wg = wg; ra.forced = forced_expert; ra.T = d.T; ra.H = d.H; ra.E = d.E; ra.C = d.C;
  ra.K = d.K;
  ra.logits = at<float>(saved, sv.logits);
  ra.expert = at<int32_t>(saved, sv.expert);
  ra.prob = at<float>(saved, sv.prob);
  ra.gap = at<float>(saved, sv.gap);
  ra.slot = at<int32_t>(saved, sv.slot);
  ra.count = at<int32_t>(saved, sv.count);
  ra.load = at<int32_t>(saved, sv.load);
  ra.tok_of = at<int32_t>(saved, sv.tok_of);
  ra.local_rank = at<int32_t>(c->scratch, sc.local_rank);
  ra.block_hist = at<int32_t>(c->scratch, sc.block_hist);
  ra.tile_ties = at<int32_t>(c->scratch, sc.tile_ties);
  ra.ties = at<int32_t>(saved, sv.ties);
  ra.rts = d.rts ? 1 : 0;
  ra.seed = c->priority_seed;
  ra.aux_coef = d.aux_coef;
  ra.aux_partial = d.aux ? at<float>(c->scratch, sc.auxp) : nullptr;
  ra.aux_out = d.aux ? at<float>(saved, sv.aux) : nullptr;
  {
    Scope sc_(c, MOE_K_ROUTE, st, (d.K == 1 && !d.rts ? 2 : 3) + (d.aux ? 2 : 0));
    CUDA_TRY(c, route(ra, st));
  }

  // ring slot of the peer windows used by this forward (the same on every rank: every
  // rank issues the same sequence of forwards on the communicator)
  moe_comm* m = c->comm;
  const int rslot = m ? (int)(m->gen % (uint64_t)m->plan.depth) : 0;
  const uint64_t mygen = m ? ++m->gen : 0;
  TRY(forward_core(c, x, w1, w2, y, saved, st, 0, rslot));
  if (d.ckpt && c->replayed == saved) c->replayed = nullptr;  // G/A in scratch are stale now
  c->saved_written.insert(saved);
  c->saved_slot[saved] = {rslot, mygen};
  if (m && d.peer) m->ring_gen[rslot] = mygen;
  c->last_saved = saved;
  c->last_stream = st;
  return MOE_OK;
}

moe_status moe_backward(moe_ctx* c, const void* dy, const void* saved, const void* x,
                        const float* wg, const void* w1, const void* w2, void* dx, float* dwg,
                        void* dw1, void* dw2, void* stream) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (c->poisoned) return fail(MOE_ERR_STATE, "ctx poisoned by an earlier CUDA/NCCL failure");
  if (c->comm) TRY(check_comm(c));
  if (!dy || !saved || !x || !wg || !w1 || !w2 || !dx || !dwg || !dw1 || !dw2)
    return fail(MOE_ERR_ARG, "null tensor pointer");
  if (!c->saved_written.count(saved))
    return fail(MOE_ERR_STATE, "saved blob was not written by moe_forward on this ctx");
  int rslot = 0;
  if (c->d.ckpt && c->replayed != saved)
    return fail(MOE_ERR_STATE, "checkpointed forward: call moe_forward_replay on this saved blob first");
  if (c->d.peer && !c->d.ckpt) {
    const auto it = c->saved_slot.find(saved);
    if (it == c->saved_slot.end() || c->comm->ring_gen[it->second.first] != it->second.second)
      return fail(MOE_ERR_STATE, "saved blob's peer window was reused: ring_depth or more newer forwards "
                                 "ran on the communicator before this backward");
    rslot = it->second.first;
  }
  if (!aligned16(dy) || !aligned16(x) || !aligned16(wg) || !aligned16(w1) || !aligned16(w2) ||
      !aligned16(dx) || !aligned16(dwg) || !aligned16(dw1) || !aligned16(dw2))
    return fail(MOE_ERR_ALIGN, "tensor pointers must be 16-byte aligned");
  const Dims& d = c->d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const SavedLayout& sv = c->sv;
  const ScratchLayout& sc = c->sc;
  const SlotSpace ss = slot_space(d);
  const bool solo = d.world == 1;
  const int lo = d.dtd ? d.t : 0, hi = d.dtd ? d.t + 1 : d.Gt;
  const int32_t* expert = at<int32_t>(saved, sv.expert);
  const int32_t* slot = at<int32_t>(saved, sv.slot);
  const float* prob = at<float>(saved, sv.prob);
  const float* logits = at<float>(saved, sv.logits);
  const int32_t* count = at<int32_t>(saved, sv.count);
  const bool win_xo = d.peer && !d.ckpt;  // X/O in the ring windows (else saved / CAC stash)
  const void* X = win_xo ? c->comm->win[c->comm->wx(rslot)] : at<uint8_t>(saved, sv.X);
  const void* G = d.ckpt ? at<uint8_t>(c->scratch, sc.Grec) : at<uint8_t>(saved, sv.G);
  const void* A = d.ckpt ? at<uint8_t>(c->scratch, sc.Arec) : at<uint8_t>(saved, sv.A);
  const void* O = win_xo ? c->comm->win[c->comm->wo(rslot)] : at<uint8_t>(saved, sv.O);
  float* dp = at<float>(c->scratch, sc.dp);
  void* dY = d.peer ? c->comm->win[moe_comm::W_DY] : at<uint8_t>(c->scratch, sc.dY);
  void* dO = at<uint8_t>(c->scratch, sc.dO);
  void* dH = at<uint8_t>(c->scratch, sc.dH);
  void* dXp = d.peer && d.Gt > 1 ? c->comm->win[moe_comm::W_DXP] : at<uint8_t>(c->scratch, sc.dXp);
  void* dS = d.peer ? c->comm->win[moe_comm::W_DS] : at<uint8_t>(c->scratch, sc.dS);

  // One GPU, top-1, no aux loss: B5's epilogue adds B10's gate term and writes dx rows
  // directly (no dXp round trip, no separate dx gather); dl and the extension operands
  // come from the combine-backward launch.
  const bool fused_dx = solo && d.K == 1 && !d.aux && d.E <= 16 && !c->no_fused_dx;
  // B1 combine-bwd (DTD: only this rank's slice of dO), B2 a2a, B3 all-gather
  const bool split = d.peer && d.Gt == 1 && d.Gep > 1 && c->overlap;  // as in forward_core
  uint32_t sig = 0;
  if (split) {
    SplitDst sd{dY, dO, d.ep, d.El, d.Gep};
    {
      Scope sc_(c, MOE_K_COMBINE_BWD, st, 1);
      CUDA_TRY(c, combine_bwd_split(dy, O, expert, slot, prob, count, ss, d.T, dp, sd, st));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[3], st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[3], 0));
    {
      Scope sx_(c, MOE_K_XFER, c->side, 0);
      TRY(exchange_ce_dispatch_sig(c, dO, moe_comm::W_DY, c->side, &sig));
    }
    ledger(c, MOE_COLL_A2A, 1, c->disp_bytes[1]);
  } else if (d.peer) {
    {
      Scope sc_(c, MOE_K_COMBINE_BWD, st, 2);
      CUDA_TRY(c, combine_bwd_peer(dy, O, expert, slot, prob, count, nullptr, ss, d.T, lo, hi, dp,
                                   peer_dst(c, moe_comm::W_DY), st));
    }
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(publish(c, true, 1, st));
    if (d.nvls && !d.nvls_direct) TRY(nvls_allgather(c, moe_comm::W_DY, true, 1, st));
  } else if (fused_dx) {
    // B1 + the head of B10 in one launch (dl, extension operands, dropped rows)
    Scope sc_(c, MOE_K_COMBINE_BWD, st, 1);
    CUDA_TRY(c, combine_bwd_gate(dy, O, expert, slot, prob, logits, at<int32_t>(saved, sv.tok_of), count, wg,
                                 d.T, d.H, d.E, d.C, dO, at<float>(c->scratch, sc.dl),
                                 at<uint8_t>(c->scratch, sc.aext), at<uint8_t>(c->scratch, sc.bext), dx,
                                 at<int32_t>(c->scratch, sc.dwgc), st));
  } else {
    Scope sc_(c, MOE_K_COMBINE_BWD, st, 2);
    CUDA_TRY(c, combine_bwd(dy, O, expert, slot, prob, count, ss, d.T, lo, hi, dp, dO, st));
  }
  if (!solo && !d.peer) {
    Scope sc_(c, MOE_K_COMM, st, 0);
    {
      TRY(ep_exchange(c, 0, 1, dO, dY, lo, hi, st));
      if (d.dtd) TRY(ag_expert(c, 1, dY, st));
    }
  }
  // B4 dHpre = (dY W2) * G; B5 dXpart = dHpre W1; B6 dW2 = dY^T A, dW1 = dHpre^T X
  GemmArgs g4{d.El, (int)d.R, d.Fl, d.H, dY, 0, w2, 1, dH, EPI_DGELU, const_cast<void*>(G)};
  if (split) {
    TRY(gemm_sources(c, g4, sig, d.H, d.Fl, st));
  } else {
    TRY(gemm(c, g4, st));
  }
  GemmArgs g5{d.El, (int)d.R, d.H, d.Fl, dH, 0, w1, 1, dXp, EPI_STORE, nullptr};
  GateDxArgs gdx{at<int32_t>(saved, sv.tok_of), count, at<float>(c->scratch, sc.dl), wg, d.E, d.C, dx,
                 nullptr, at<uint8_t>(c->scratch, sc.aext), at<uint8_t>(c->scratch, sc.bext)};
  if (fused_dx) {
    g5.epilogue = EPI_SCATTER;
    g5.gdx = &gdx;
  }
  // (G_t = 1, split exchange) B5 + B8 fused: dX rows straight into the source ranks' dS
  // windows from B5's epilogue (as F7 + F9 in the forward)
  const bool fused_ret = split && !c->no_fused_return;
  PeerOut po;
  if (fused_ret) {
    po.table = c->comm->d_table;
    po.nwin = c->comm->nwin;
    po.win = moe_comm::W_DS;
    po.rank0 = d.d * d.Gep;
    po.e0 = d.ep * d.El;
    po.C = d.C;
    g5.po = &po;
  }
  TRY(gemm(c, g5, st));
  GemmArgs g6{d.El, d.H, d.Fl, (int)d.R, dY, 1, A, 1, dw2, EPI_STORE, nullptr};
  GemmArgs g7{d.El, d.Fl, d.H, (int)d.R, dH, 1, X, 1, dw1, EPI_STORE, nullptr};
  if (fused_ret) {
    TRY(gemm(c, g6, st));
    TRY(gemm(c, g7, st));
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(barrier(c, st));  // every rank's B5 rows are in the dS windows
    if (d.Gep > 1) ledger(c, MOE_COLL_A2A, 1, c->ret_bytes[1]);
    if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, 1, c->ret_bytes[2]);
  } else if (d.peer && d.Gt > 1) {
    // B7-B9 fused over peer memory (tp_return), then the weight-gradient GEMMs
    {
      Scope sc_(c, MOE_K_COMM, st, 0);
      TRY(barrier(c, st));  // every TP partial of dX complete
      ReduceReturn rr;
      rr.table = c->comm->d_table;
      rr.nwin = c->comm->nwin;
      rr.src_win = moe_comm::W_DXP;
      rr.dst_win = moe_comm::W_DS;
      rr.d = d.d; rr.ep = d.ep; rr.t = d.t; rr.Gt = d.Gt; rr.Gep = d.Gep; rr.El = d.El; rr.E = d.E;
      rr.H = d.H; rr.Cs = d.Cs; rr.dtd = d.dtd ? 1 : 0;
      rr.fold = d.dtd && (!d.nvls || d.nvls_direct) ? 1 : 0;
      rr.mc = d.nvls_direct && !c->comm->mcwin.empty() ? c->comm->mcwin[moe_comm::W_DS] : nullptr;
      CUDA_TRY(c, reduce_return(rr, st));
      c->stats.kernel_launches[MOE_K_COMM] += 1;
    }
    TRY(gemm(c, g6, st));
    TRY(gemm(c, g7, st));
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(barrier(c, st));  // every destination written (each rank's reduce precedes its barrier)
    const int64_t xe = (int64_t)d.El * d.R * d.H * 2;
    if (d.dtd) ledger(c, MOE_COLL_REDUCESCATTER, 1, xe * (d.Gt - 1) / d.Gt);
    else ledger(c, MOE_COLL_ALLREDUCE, 1, 2 * xe * (d.Gt - 1) / d.Gt);
    if (d.Gep > 1) ledger(c, MOE_COLL_A2A, 1, c->ret_bytes[1]);
    if (d.nvls && !d.nvls_direct) TRY(nvls_allgather(c, moe_comm::W_DS, false, 1, st));
    else if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, 1, ag_bytes(d, c->ret_bytes[2]));
  } else if (d.peer) {
    // B7-B9 (TP reduction + return pieces) on the side stream, overlapping the
    // weight-gradient GEMMs, which do not feed them
    CUDA_TRY(c, cudaEventRecord(c->ev[0], st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[0], 0));
    if (!c->overlap) {
      TRY(gemm(c, g6, st));
      TRY(gemm(c, g7, st));
      CUDA_TRY(c, cudaEventRecord(c->ev[0], st));
      CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[0], 0));
    }
    if (d.Gt > 1) {
      if (d.dtd) TRY(rs_expert(c, 1, dXp, c->side));
      else TRY(ar_expert(c, 1, dXp, c->side));
    }
    {
      Scope sx_(c, MOE_K_XFER, c->side, 0);
      TRY(exchange_ce(c, dXp, moe_comm::W_DS, 0, d.El, c->side));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[1], c->side));
    if (c->overlap) {
      TRY(gemm(c, g6, st));
      TRY(gemm(c, g7, st));
    }
    Scope sc_(c, MOE_K_COMM, st, 0);
    TRY(exchange_local(c, dXp, moe_comm::W_DS, st));  // own pieces: need only B5's output
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev[1], 0));
    TRY(barrier(c, st));
    if (d.Gep > 1) ledger(c, MOE_COLL_A2A, 1, c->ret_bytes[1]);
    if (d.dtd) ledger(c, MOE_COLL_ALLGATHER, 1, c->ret_bytes[2]);
  } else {
    TRY(gemm(c, g6, st));
    TRY(gemm(c, g7, st));
    // B7 TP reduce, B8 a2a back, B9 all-gather
    if (!solo) {
      Scope sc_(c, MOE_K_COMM, st, 0);
      if (d.Gt > 1) {
        if (d.dtd) TRY(rs_expert(c, 1, dXp, st));
        else TRY(ar_expert(c, 1, dXp, st));
      }
      TRY(ep_exchange(c, 1, 1, dS, dXp, lo, hi, st));
      if (d.dtd) TRY(ag_slot(c, 1, dS, st));
    }
  }
  // B10 dispatch-bwd + gate-bwd (fused path: only dWg is left)
  if (fused_dx) {
    // dWg = X^T a_ext over the kept slot rows (dl = 0 for dropped tokens)
    Scope sc_(c, MOE_K_GATE_BWD, st, 1);
    CUDA_TRY(c, gate_dwg_tc(X, at<uint8_t>(c->scratch, sc.aext), (int64_t)d.E * d.C, d.H, d.E, dwg,
                            at<float>(c->scratch, sc.dwgp), DWG_TC_SPLITS, at<int32_t>(c->scratch, sc.dwgc), st));
  } else {
    Scope sc_(c, MOE_K_GATE_BWD, st, d.E <= 32 ? 4 : 5);
    CUDA_TRY(c, gate_bwd(x, dS, wg, logits, expert, slot, prob, dp, ss, d.T, dx, dwg,
                         at<float>(c->scratch, sc.dl), at<int32_t>(c->scratch, sc.grow),
                         at<float>(c->scratch, sc.dwgp), sc.nsplit,
                         at<uint8_t>(c->scratch, sc.wpk), at<uint8_t>(c->scratch, sc.atok),
                         at<int32_t>(c->scratch, sc.dwgc),
                         d.aux ? at<const float>(saved, sv.aux) : nullptr, d.aux_coef, st));
  }
  c->last_stream = st;
  return MOE_OK;
}

moe_status moe_forward_replay(moe_ctx* c, const void* saved, const void* x, const float* wg,
                              const void* w1, const void* w2, void* stream) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (c->poisoned) return fail(MOE_ERR_STATE, "ctx poisoned by an earlier CUDA/NCCL failure");
  if (c->comm) TRY(check_comm(c));
  if (!c->d.ckpt) return fail(MOE_ERR_STATE, "moe_forward_replay needs MOE_F_CHECKPOINT");
  if (!saved || !x || !wg || !w1 || !w2) return fail(MOE_ERR_ARG, "null tensor pointer");
  if (!c->saved_written.count(saved))
    return fail(MOE_ERR_STATE, "saved blob was not written by moe_forward on this ctx");
  const Dims& d = c->d;
  const SavedLayout& sv = c->sv;
  const ScratchLayout& sc = c->sc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* sv_mut = const_cast<void*>(saved);
  if (d.cac) {
    // CAC: the stashed output of the first collective (X) feeds
    // GEMM1 directly; no gate, no dispatch, no collective is re-issued.
    GemmArgs g1{d.El, (int)d.R, d.Fl, d.H, at<uint8_t>(sv_mut, sv.X), 0, w1, 0,
                at<uint8_t>(c->scratch, sc.Grec), EPI_GELU, at<uint8_t>(c->scratch, sc.Arec)};
    TRY(gemm(c, g1, st));
  } else {
    // plain activation checkpointing: the whole forward again (routing record reused:
    // it is deterministic and needs no communication), every collective re-issued
    moe_comm* m = c->comm;
    const int rslot = m ? (int)(m->gen % (uint64_t)m->plan.depth) : 0;
    if (m) {
      const uint64_t g = ++m->gen;
      if (d.peer) m->ring_gen[rslot] = g;
    }
    TRY(forward_core(c, x, w1, w2, nullptr, sv_mut, st, 2, rslot));
  }
  (void)wg;
  c->replayed = saved;
  c->last_stream = st;
  return MOE_OK;
}

moe_status moe_routing(moe_ctx* c, const void* saved, int32_t* expert, int32_t* slot, float* prob,
                       float* gap, int32_t* count, void* stream) {
  if (!c || !saved) return fail(MOE_ERR_ARG, "null ctx/saved");
  if (!c->saved_written.count(saved)) return fail(MOE_ERR_STATE, "saved blob not written by this ctx");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims& d = c->d;
  const SavedLayout& sv = c->sv;
  auto cp = [&](void* dst, size_t off, size_t bytes) -> moe_status {
    if (!dst) return MOE_OK;
    CUDA_TRY(c, cudaMemcpyAsync(dst, at<uint8_t>(saved, off), bytes, cudaMemcpyDeviceToDevice, st));
    return MOE_OK;
  };
  TRY(cp(expert, sv.expert, (size_t)d.T * d.K * 4));
  TRY(cp(slot, sv.slot, (size_t)d.T * d.K * 4));
  TRY(cp(prob, sv.prob, (size_t)d.T * d.K * 4));
  TRY(cp(gap, sv.gap, (size_t)d.T * 4));
  TRY(cp(count, sv.count, (size_t)d.E * 4));
  return MOE_OK;
}

moe_status moe_aux_loss(moe_ctx* c, const void* saved, float* aux, void* stream) {
  if (!c || !saved || !aux) return fail(MOE_ERR_ARG, "null ctx/saved/output");
  if (!c->d.aux) return fail(MOE_ERR_STATE, "MOE_F_AUX_LOSS not set");
  if (!c->saved_written.count(saved)) return fail(MOE_ERR_STATE, "saved blob not written by this ctx");
  CUDA_TRY(c, cudaMemcpyAsync(aux, at<uint8_t>(saved, c->sv.aux + 4 * (size_t)c->d.E), 4,
                              cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return MOE_OK;
}

moe_status moe_set_priority_seed(moe_ctx* c, uint64_t seed) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  c->priority_seed = seed;
  return MOE_OK;
}

moe_status moe_stats_get(moe_ctx* c, moe_stats* out) {
  if (!c || !out) return fail(MOE_ERR_ARG, "null ctx/output");
  if (c->last_stream) CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  if (c->last_saved) {
    int32_t ties = 0;
    std::vector<int32_t> count(c->d.E);
    CUDA_TRY(c, cudaMemcpy(&ties, at<uint8_t>(c->last_saved, c->sv.ties), 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(c, cudaMemcpy(count.data(), at<uint8_t>(c->last_saved, c->sv.count), 4 * c->d.E,
                           cudaMemcpyDeviceToHost));
    int64_t kept = 0;
    for (int32_t v : count) kept += v;
    c->stats.tie_tokens = ties;
    c->stats.dropped_tokens = c->d.T * c->d.K - kept;  // dropped (token, choice) pairs
  }
  for (auto& sp : c->spans) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) c->stats.kernel_ms[sp.cls] += ms;
    c->pool.push_back(sp.a);
    c->pool.push_back(sp.b);
  }
  c->spans.clear();
  c->stats.nccl_async_error = 0;
  ncclComm_t comms[3] = {c->comm ? c->comm->world_comm : nullptr, c->comm ? c->comm->tp_comm : nullptr,
                         c->comm ? c->comm->ep_comm : nullptr};
  for (ncclComm_t m : comms) {
    if (!m) continue;
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(m, &ae) == ncclSuccess && ae != ncclSuccess) c->stats.nccl_async_error = (int)ae;
  }
  *out = c->stats;
  if (c->comm) return check_comm(c);
  return MOE_OK;
}

moe_status moe_stats_reset(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  std::memset(&c->stats, 0, sizeof(c->stats));
  return MOE_OK;
}

moe_status moe_set_timing(moe_ctx* c, int on) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (!(c->cfg.flags & MOE_F_TIMING)) return fail(MOE_ERR_STATE, "moe_set_timing needs MOE_F_TIMING");
  c->timing = on != 0;
  return MOE_OK;
}

moe_status moe_gemm_bf16(int batch, int M, int N, int K, const void* A, int a_mn, const void* B,
                         int b_mn, void* D, int epilogue, void* aux, int impl, void* stream) {
  if (batch < 0 || M < 0 || N < 0 || K < 0) return fail(MOE_ERR_ARG, "negative size");
  if (!A || !B || !D) return fail(MOE_ERR_ARG, "null operand");
  if (epilogue < 0 || epilogue > 2) return fail(MOE_ERR_ARG, "bad epilogue");
  if (epilogue != EPI_STORE && !aux) return fail(MOE_ERR_ARG, "epilogue needs aux");
  if (N % 64 || M % 8 || K % 8) return fail(MOE_ERR_SHAPE, "need N % 64 == 0, M % 8 == 0, K % 8 == 0");
  if (!aligned16(A) || !aligned16(B) || !aligned16(D) || (aux && !aligned16(aux)))
    return fail(MOE_ERR_ALIGN, "operands must be 16-byte aligned");
  GemmArgs g{batch, M, N, K, A, a_mn ? 1 : 0, B, b_mn ? 1 : 0, D, epilogue, aux};
  if (impl != 0 && impl != 1) return fail(MOE_ERR_UNSUPPORTED, "impl must be 0 (tcgen05) or 1 (SIMT reference)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (impl == 1) {
    cudaError_t e = gemm_ref(g, st);
    if (e != cudaSuccess) return fail(MOE_ERR_CUDA, cudaGetErrorString(e));
    return MOE_OK;
  }
  return gemm(nullptr, g, st);
}

moe_status moe_adamw_plan(int64_t n, int64_t tile_params, int64_t* n_tiles, size_t* temp_bytes) {
  if (n < 0 || tile_params < 0 || !n_tiles || !temp_bytes) return fail(MOE_ERR_ARG, "bad arguments");
  if (tile_params == 0) {
    *n_tiles = n > 0 ? 1 : 0;
    *temp_bytes = 0;
  } else {
    *n_tiles = (n + tile_params - 1) / tile_params;
    *temp_bytes = 4 * (size_t)(n < tile_params ? n : tile_params);
  }
  return MOE_OK;
}

moe_status moe_adamw_step(const void* grad, float* master, float* exp_avg, float* exp_avg_sq,
                          void* param, int64_t n, const moe_adamw_hparams* h, int64_t tile_params,
                          float* temp, void* stream) {
  if (!h || n < 0 || tile_params < 0) return fail(MOE_ERR_ARG, "bad arguments");
  if (h->step < 1) return fail(MOE_ERR_ARG, "step must be >= 1");
  if (n == 0) return MOE_OK;
  if (!grad || !master || !exp_avg || !exp_avg_sq) return fail(MOE_ERR_ARG, "null array");
  if (tile_params > 0 && !temp) return fail(MOE_ERR_ARG, "tiled step needs temp (moe_adamw_plan)");
  if (tile_params == 0 && temp) return fail(MOE_ERR_ARG, "fused step takes no temp");
  if (!aligned16(grad) || !aligned16(master) || !aligned16(exp_avg) || !aligned16(exp_avg_sq) ||
      (param && !aligned16(param)) || (temp && !aligned16(temp)))
    return fail(MOE_ERR_ALIGN, "arrays must be 16-byte aligned");
  // per-step scalars: binary64, rounded once to binary32 (reading R19)
  const double c1 = 1.0 - std::pow(h->beta1, (double)h->step);
  const double c2 = 1.0 - std::pow(h->beta2, (double)h->step);
  AdamwScalars s;
  s.b1 = (float)h->beta1;
  s.b2 = (float)h->beta2;
  s.ob1 = (float)(1.0 - h->beta1);
  s.ob2 = (float)(1.0 - h->beta2);
  s.step = (float)(h->lr / c1);
  s.c2s = (float)std::sqrt(c2);
  s.decay = (float)(1.0 - h->lr * h->weight_decay);
  s.eps = (float)h->eps;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (tile_params == 0) {
    e = adamw_fused(grad, master, exp_avg, exp_avg_sq, param, n, s, st);
  } else {
    int launches = 0;
    e = adamw_tiled(grad, master, exp_avg, exp_avg_sq, param, n, s, tile_params, temp, st, &launches);
  }
  if (e != cudaSuccess) return fail(MOE_ERR_CUDA, std::string("adamw: ") + cudaGetErrorString(e));
  return MOE_OK;
}

}  // extern "C"
