// plan.h — derived dimensions, buffer layouts and the collective schedule.
// Pure host code (no CUDA calls) so the CPU tests can check it without a GPU.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/moe.h"

namespace moe {

struct Dims {
  int64_t T;
  int H, F, E;
  int Gt, Gep, Gd, world, rank;
  int d, ep, t;
  int El, Fl;
  int64_t C, Cs, R;  // capacity, slot slice, rows per local expert
  int S;             // token groups
  bool dtd;          // DTD in effect (requested and G_t > 1)
  bool forced;
  bool peer;         // world > 1 and the peer-memory exchange (not MOE_F_NCCL_EXCHANGE)
  bool nvls;         // MOE_F_NVLS with DTD in effect
  bool nvls_direct;  //   G_ep == 1: every destination is the own TP group -> the fused exchange
                     //   kernels store once through the multicast mapping (no extra step);
                     //   else: a2a of the own slice, then a multicast all-gather step
  bool ckpt;         // MOE_F_CHECKPOINT
  bool cac;          // MOE_F_CAC (with ckpt)
  bool rts;          // MOE_F_RANDOM_PRIORITY
  bool aux;          // MOE_F_AUX_LOSS
  float aux_coef;
  int K;             // experts per token (top_k: 1 or 2)
  int ring_depth;    // forwards in flight per communicator (peer windows of X, O)
  int64_t timeout_ms;  // deadline of a peer barrier / signal wait
};

// Validates and derives; returns MOE_OK or an error with *why set.
moe_status make_dims(const moe_config* cfg, int world, int rank, Dims* d, std::string* why);

struct SavedLayout {
  size_t logits, expert, slot, prob, gap, count, load, ties, tok_of, aux, X, G, A, O, total;  // G = gelu'(Hpre)
};
struct ScratchLayout {
  // forward
  size_t local_rank, block_hist, tile_ties, auxp, D, Ypart;
  // backward
  size_t dp, dl, grow, atok, dwgp, dwgc, wpk, dO, dY, dH, dXp, dS, aext, bext;
  // checkpoint mode: G, A re-materialized by the replay (outside both regions)
  size_t Grec, Arec;
  size_t total;
  bool D_in_saved, Y_in_saved;  // world == 1: D aliases saved.X, Ypart aliases saved.O
  bool dO_is_dY, dXp_is_dS;     // world == 1: slot space == expert space
  int nsplit;
};

void make_layouts(const Dims& d, SavedLayout* sv, ScratchLayout* sc);

// Collective schedule of one forward + backward on this rank (issue order).
std::vector<moe_collective> make_schedule(const Dims& d);

}  // namespace moe
