// plan.cpp — host-only planning: validation (moe.h constraints), the HBM
// layout of the saved/scratch blobs and the collective schedule/ledger.
#include "plan.h"

#include <cmath>

#include "internal.h"

namespace moe {

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

moe_status make_dims(const moe_config* c, int world, int rank, Dims* d, std::string* why) {
  if (!c || !d) { *why = "null config/output"; return MOE_ERR_ARG; }
  if (world < 1 || rank < 0 || rank >= world) { *why = "rank/world out of range"; return MOE_ERR_ARG; }
  if (c->tokens < 1 || c->hidden < 1 || c->ffn < 1 || c->experts < 1 || c->g_tensor < 1 ||
      c->g_expert < 1 || !(c->capacity_factor > 0.f) || !std::isfinite(c->capacity_factor)) {
    *why = "tokens, hidden, ffn, experts, g_tensor, g_expert and capacity_factor must be positive";
    return MOE_ERR_ARG;
  }
  if (c->experts > 64) { *why = "experts must be <= 64"; return MOE_ERR_SHAPE; }
  if (c->hidden % 64) { *why = "hidden % 64 != 0"; return MOE_ERR_SHAPE; }
  if (c->ffn % c->g_tensor) { *why = "ffn % g_tensor != 0"; return MOE_ERR_SHAPE; }
  if ((c->ffn / c->g_tensor) % 64) { *why = "(ffn / g_tensor) % 64 != 0"; return MOE_ERR_SHAPE; }
  if (c->experts % c->g_expert) { *why = "experts % g_expert != 0"; return MOE_ERR_SHAPE; }
  const int tp_ep = c->g_tensor * c->g_expert;
  if (world % tp_ep) { *why = "world % (g_tensor * g_expert) != 0"; return MOE_ERR_SHAPE; }
  if (c->tokens > (int64_t)1 << 30) { *why = "tokens must be < 2^30"; return MOE_ERR_SHAPE; }
  if (c->flags & ~(MOE_F_STATS | MOE_F_FORCED_ROUTING | MOE_F_TIMING | MOE_F_NCCL_EXCHANGE |
                   MOE_F_CHECKPOINT | MOE_F_CAC | MOE_F_RANDOM_PRIORITY | MOE_F_AUX_LOSS | MOE_F_NVLS)) {
    *why = "unknown flag bits";
    return MOE_ERR_ARG;
  }
  if ((c->flags & MOE_F_AUX_LOSS) && !(c->aux_loss_coef >= 0.f && std::isfinite(c->aux_loss_coef))) {
    *why = "aux_loss_coef must be finite and >= 0";
    return MOE_ERR_ARG;
  }
  if (c->top_k < 0 || c->top_k > 2) { *why = "top_k must be 0, 1 or 2"; return MOE_ERR_ARG; }
  if (c->top_k == 2 && c->experts < 2) { *why = "top-2 needs experts >= 2"; return MOE_ERR_SHAPE; }
  if (c->top_k == 2 && (c->flags & MOE_F_FORCED_ROUTING)) {
    *why = "forced routing is top-1 only";
    return MOE_ERR_UNSUPPORTED;
  }
  d->K = c->top_k == 2 ? 2 : 1;
  d->T = c->tokens;
  d->H = c->hidden;
  d->F = c->ffn;
  d->E = c->experts;
  d->Gt = c->g_tensor;
  d->Gep = c->g_expert;
  d->Gd = world / tp_ep;
  d->world = world;
  d->rank = rank;
  d->t = rank % d->Gt;
  d->ep = (rank / d->Gt) % d->Gep;
  d->d = rank / tp_ep;
  d->El = d->E / d->Gep;
  d->Fl = d->F / d->Gt;
  // Reading R2: C = ceil(cf*K*T/E) (double), >= 1, rounded up to a multiple of G_t (R22: K = 2).
  int64_t C = (int64_t)std::ceil((double)c->capacity_factor * (double)d->K * (double)d->T / (double)d->E);
  if (C < 1) C = 1;
  C = ceil_div(C, d->Gt) * d->Gt;
  d->C = C;
  d->Cs = C / d->Gt;
  d->R = (int64_t)d->Gep * C;
  d->S = world / d->Gt;
  d->dtd = c->dtd != 0 && d->Gt > 1;
  d->forced = (c->flags & MOE_F_FORCED_ROUTING) != 0;
  d->peer = world > 1 && (c->flags & MOE_F_NCCL_EXCHANGE) == 0;
  d->nvls = (c->flags & MOE_F_NVLS) != 0 && d->peer && d->dtd;
  d->nvls_direct = d->nvls && d->Gep == 1;
  d->ckpt = (c->flags & MOE_F_CHECKPOINT) != 0;
  d->cac = d->ckpt && (c->flags & MOE_F_CAC) != 0;
  d->rts = (c->flags & MOE_F_RANDOM_PRIORITY) != 0;
  d->aux = (c->flags & MOE_F_AUX_LOSS) != 0;
  d->aux_coef = d->aux ? c->aux_loss_coef : 0.f;
  if ((c->flags & MOE_F_CAC) && !d->ckpt) { *why = "MOE_F_CAC needs MOE_F_CHECKPOINT"; return MOE_ERR_ARG; }
  if (d->R > (int64_t)1 << 30) { *why = "rows per expert too large"; return MOE_ERR_SHAPE; }
  if (c->ring_depth < 0 || c->ring_depth > 64) { *why = "ring_depth must be in [0, 64]"; return MOE_ERR_ARG; }
  if (c->peer_timeout_ms < 0) { *why = "peer_timeout_ms must be >= 0"; return MOE_ERR_ARG; }
  d->ring_depth = c->ring_depth ? c->ring_depth : 2;
  d->timeout_ms = c->peer_timeout_ms ? c->peer_timeout_ms : 60000;
  if (d->peer && d->dtd && d->Gt > 8) {
    // the fused peer dispatch / combine-backward resolve at most 8 destination rows per slot
    *why = "the peer-memory exchange supports DTD with g_tensor <= 8 (use MOE_F_NCCL_EXCHANGE)";
    return MOE_ERR_UNSUPPORTED;
  }
  return MOE_OK;
}

namespace {
struct Bump {
  size_t off = 0;
  size_t take(size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  }
};
}  // namespace

void make_layouts(const Dims& d, SavedLayout* sv, ScratchLayout* sc) {
  const size_t slot_space = (size_t)d.E * d.C * d.H * 2;            // [G_t][E][C_s][H]
  const size_t expert_space = (size_t)d.El * d.R * d.H * 2;         // [E_l][R][H]
  const size_t ffn_space = (size_t)d.El * d.R * d.Fl * 2;           // [E_l][R][F_l]
  Bump s;
  sv->logits = s.take((size_t)d.T * d.E * 4);
  sv->expert = s.take((size_t)d.T * d.K * 4);
  sv->slot = s.take((size_t)d.T * d.K * 4);
  sv->prob = s.take((size_t)d.T * d.K * 4);
  sv->gap = s.take((size_t)d.T * 4);
  sv->count = s.take((size_t)d.E * 4);
  sv->load = s.take((size_t)d.E * 4);
  sv->ties = s.take(4);
  sv->tok_of = s.take((size_t)d.E * d.C * 4);
  sv->aux = d.aux ? s.take((size_t)(d.E + 1) * 4) : 0;  // f_e [E], then l_aux
  // peer mode keeps X and O in the library's ring windows instead of the saved blob,
  // except under checkpointing, where they are the CAC stash; checkpointing keeps G/A
  // out of the saved blob (the replay re-materializes them in scratch)
  sv->X = (d.peer && !d.ckpt) ? 0 : s.take(expert_space);
  sv->G = d.ckpt ? 0 : s.take(ffn_space);
  sv->A = d.ckpt ? 0 : s.take(ffn_space);
  sv->O = (d.peer && !d.ckpt) ? 0 : s.take(slot_space);
  sv->total = s.off;

  const bool solo = d.world == 1;  // slot space == expert space, no communication
  sc->D_in_saved = solo;
  sc->Y_in_saved = solo;
  sc->dO_is_dY = solo;
  sc->dXp_is_dS = solo;
  sc->nsplit = gate_bwd_splits(d.T);
  Bump f;
  sc->local_rank = f.take((size_t)d.T * d.K * 4);
  // gate tiles hold R >= 8 tokens (route.cu), 1024-item blocks for the unfused scan
  sc->block_hist = f.take((size_t)((d.T * d.K + 7) / 8) * d.E * 4);
  sc->tile_ties = f.take((size_t)((d.T + 7) / 8) * 4);
  sc->auxp = d.aux ? f.take((size_t)AUX_GRID * d.E * 8) : 0;  // P partials + first-choice counts
  // peer mode dispatches straight into windows; with G_t = 1 (split exchange) the rows of
  // remote experts are staged in slot space for the copy engines
  const bool split = d.peer && d.Gt == 1 && d.Gep > 1;
  sc->D = solo ? 0 : (d.peer ? (split ? f.take(slot_space) : 0) : f.take(slot_space));
  sc->Ypart = solo ? 0 : f.take(expert_space);
  Bump b;  // backward region reuses the forward region
  sc->dp = b.take((size_t)d.T * d.K * 4);
  sc->dl = b.take((size_t)d.T * d.E * 4);
  sc->grow = b.take((size_t)d.T * d.K * 4);  // gathered slot-space rows of the general B10
  sc->atok = b.take((size_t)d.T * 64 * 2);     // its [hi | lo](dl) rows for the tcgen05 dWg
  sc->dwgp = b.take((size_t)(sc->nsplit > DWG_TC_SPLITS ? sc->nsplit : DWG_TC_SPLITS) * d.H * d.E * 4);
  sc->dwgc = b.take((size_t)((d.H + 127) / 128) * 4);  // split-K counters of the one-GPU dWg launch
  sc->wpk = b.take(gate_bwd_pack_bytes(d.H, d.E));
  sc->aext = solo ? b.take((size_t)d.E * d.C * 64 * 2) : 0;  // one-GPU fused B5 + B10 (K extension)
  sc->bext = solo ? b.take((size_t)64 * d.H * 2) : 0;
  sc->dY = d.peer ? 0 : b.take(expert_space);   // peer mode: window WdY
  sc->dO = solo ? sc->dY : (d.peer ? (split ? b.take(slot_space) : 0) : b.take(slot_space));
  sc->dH = b.take(ffn_space);
  sc->dXp = b.take(expert_space);
  sc->dS = solo ? sc->dXp : (d.peer ? 0 : b.take(slot_space));  // peer mode: window WdS
  size_t top = f.off > b.off ? f.off : b.off;
  sc->Grec = sc->Arec = 0;
  if (d.ckpt) {
    Bump r;
    r.off = top;
    sc->Grec = r.take(ffn_space);
    sc->Arec = r.take(ffn_space);
    top = r.off;
  }
  sc->total = top;
}

std::vector<moe_collective> make_schedule(const Dims& d) {
  std::vector<moe_collective> v;
  const int64_t elt = 2;  // bf16
  const int64_t slices = d.dtd ? 1 : d.Gt;  // slot slices a rank sends per expert
  auto push = [&](int kind, int pass, int step, int gsize, int64_t buf, int64_t wire) {
    moe_collective c;
    c.kind = kind; c.pass = pass; c.step = step; c.group_size = gsize;
    c.buffer_bytes = buf; c.wire_bytes = wire;
    v.push_back(c);
  };
  const int64_t a2a_buf = (int64_t)d.E * slices * d.Cs * d.H * elt;       // send buffer incl. self
  const int64_t a2a_wire = (int64_t)(d.Gep - 1) * d.El * slices * d.Cs * d.H * elt;
  const int64_t xe = (int64_t)d.El * d.R * d.H * elt;                       // expert-space buffer
  const int64_t O = (int64_t)d.E * d.C * d.H * elt;                         // slot-space buffer
  const int64_t g = d.Gt;
  const int npass = (d.ckpt && !d.cac) ? 3 : 2;  // plain checkpointing replays the forward's collectives
  for (int pi = 0; pi < npass; ++pi) {
    const int pass = npass == 3 ? (pi == 0 ? 0 : (pi == 1 ? 2 : 1)) : pi;  // issue order
    // forward: F4 a2a, F5 AG (DTD), [GEMMs], F8 RS/AR, F9 a2a, F10 AG (DTD)
    // backward mirrors it: B2 a2a, B3 AG (DTD), [GEMMs], B7 RS/AR, B8 a2a, B9 AG (DTD)
    const bool bwd = pass == 1;  // replay (pass 2) repeats the forward steps
    const int s_a2a1 = bwd ? 2 : 4, s_ag1 = bwd ? 3 : 5, s_red = bwd ? 7 : 8;
    const int s_a2a2 = bwd ? 8 : 9, s_ag2 = bwd ? 9 : 10;
    // NVLS: a rank's all-gather egress is its own slice once (the switch replicates it)
    const int64_t ag_x = d.nvls ? xe / g : xe * (g - 1) / g, ag_o = d.nvls ? O / g : O * (g - 1) / g;
    if (d.Gep > 1) push(MOE_COLL_A2A, pass, s_a2a1, d.Gep, a2a_buf, a2a_wire);
    if (d.dtd) push(MOE_COLL_ALLGATHER, pass, s_ag1, d.Gt, xe, ag_x);
    if (d.Gt > 1) {
      if (d.dtd) push(MOE_COLL_REDUCESCATTER, pass, s_red, d.Gt, xe, xe * (g - 1) / g);
      else push(MOE_COLL_ALLREDUCE, pass, s_red, d.Gt, xe, 2 * xe * (g - 1) / g);
    }
    if (d.Gep > 1) push(MOE_COLL_A2A, pass, s_a2a2, d.Gep, a2a_buf, a2a_wire);
    if (d.dtd) push(MOE_COLL_ALLGATHER, pass, s_ag2, d.Gt, O, ag_o);
  }
  return v;
}

}  // namespace moe
