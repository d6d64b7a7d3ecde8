// internal.h — host-side declarations shared by the libmoe translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace moe {

// Batched GEMM D[b] = epi(A[b] . B[b]^T); layouts as in moe.h (moe_gemm_bf16).
enum { EPI_STORE = 0, EPI_GELU = 1, EPI_DGELU = 2, EPI_COMBINE = 4, EPI_SCATTER = 5 };

// EPI_SCATTER (B5 on one GPU, top-1, no aux loss, E <= 16): B10's gate term rides on the
// tensor cores as one extra 64-wide K block — A_ext[e][c] = [hi(dl_t) | lo(dl_t) | hi(dl_t) | 0]
// (bf16, t = tok_of[e][c], zeros for empty slots), B_ext = [hi(Wg)^T ; hi(Wg)^T ; lo(Wg)^T ; 0]
// ([64][H] bf16) — and the epilogue writes dx[tok_of[e][c]] = bf16(acc) for kept slots.
struct GateDxArgs {
  const int32_t* tok_of;  // [E][C]
  const int32_t* count;   // [E]
  const float* dl;        // [T][E]
  const float* wg;        // [H][E]
  int E;
  int64_t C;
  void* dx;               // bf16 [T][H] (EPI_COMBINE: y)
  const float* prob;      // EPI_COMBINE: [T] combine weights
  const void* a_ext;      // EPI_SCATTER: bf16 [E][C][64]
  const void* b_ext;      // EPI_SCATTER: bf16 [64][H]
};
// EPI_COMBINE (F7 on one GPU, top-1): the epilogue stores O as usual and also
// y[tok_of[e][c]] = bf16(p_t * acc) for kept slots (F11 fused; uses tok_of, count, C,
// prob and dx = y of GateDxArgs).

// Tile-completion signal (G_t = 1 return overlap): the batches [part_b[q], part_b[q+1]) form
// part q; when the last CTA finishes its share of part q's tiles (stores visible at system
// scope), flag[q] = epoch (release) — a stream waiting on that value (cuStreamWaitValue32)
// starts the part's copy-engine transfers while the same GEMM launch computes the next
// parts. cnt[q] counts CTA tile completions and is reset by the last arrival.
struct GemmSignal {
  int32_t* cnt = nullptr;  // [4], zero between launches
  uint32_t* flag = nullptr;  // [4]
  uint32_t epoch = 0;
  int nparts = 0;
  int part_b[5] = {0, 0, 0, 0, 0};
};

// Fused return exchange (G_t = 1 split mode, F7 -> F9): EPI_STORE rows of batch b (local
// expert) go straight into the slot-space window of their source rank over peer memory:
// row m of source block s = m / C lands at ((e0 + b) C + m - s C) of window `win` of rank
// rank0 + s (table: [world][nwin] window pointers, device). The GEMM's D is not written.
struct PeerOut {
  void* const* table = nullptr;
  int nwin = 0, win = 0, rank0 = 0, e0 = 0;
  int64_t C = 0;
};

struct GemmArgs {
  int batch, M, N, K;
  const void* A;
  int a_mn;  // 0: A [b][M][K]; 1: A [b][K][M]
  const void* B;
  int b_mn;  // 0: B [b][N][K]; 1: B [b][K][N]
  void* D;   // [b][M][N]
  int epilogue;
  void* aux;  // EPI_GELU: out A = gelu(acc) [b][M][N] (D = gelu'(acc)); EPI_DGELU: in G [b][M][N] (D = acc*G)
  // Batch strides in elements (0 = dense): rows [0, M) of batch b of A (K-major only)
  // start at A + b * a_bs; of D / aux at D + b * d_bs (a row block of a larger batch,
  // e.g. the rows of one source rank inside [E_l][G_ep][C]).
  int64_t a_bs = 0, d_bs = 0;
  const GateDxArgs* gdx = nullptr;  // EPI_SCATTER / EPI_COMBINE only
  const GemmSignal* sig = nullptr;  // EPI_STORE only: per-part completion flags
  const PeerOut* po = nullptr;      // EPI_STORE only: rows stored into the source ranks' windows
};

// tcgen05 / TMEM / TMA kernel (the product path).
cudaError_t gemm_tc(const GemmArgs& a, cudaStream_t s, const char** why);
// Plain SIMT kernel: bring-up cross-check only (moe_gemm_bf16 impl=1).
cudaError_t gemm_ref(const GemmArgs& a, cudaStream_t s);
// (gemm_sm100.cu) 2-D bf16 TMA map {inner, outer}, box {box_inner, box_outer}, 128B
// swizzle, into the 128-byte CUtensorMap at `map`; *sms = the device's SM count.
cudaError_t tensor_map_bf16(void* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                            uint32_t box_outer, int* sms);

// ---- routing / permutation kernels (route.cu, permute.cu) ----
constexpr int AUX_GRID = 64;
constexpr int DWG_TC_SPLITS = 16;  // most split-K partials of gate_dwg_tc  // CTAs of the deterministic P_e reduction (aux loss)
struct RouteArgs {
  const void* x;        // bf16 [T][H]
  const float* wg;      // [H][E]
  const int32_t* forced;  // [T] or null
  int64_t T;
  int H, E;
  int K;                // experts per token (1, or 2 for top-2, R22)
  int64_t C;
  float* logits;        // [T][E]
  int32_t* expert;      // [T][K]
  float* prob;          // [T][K] combine weights
  float* gap;           // [T]
  int32_t* slot;        // [T][K]
  int32_t* count;       // [E]   kept per expert
  int32_t* load;        // [E]   routed per expert (pre-capacity)
  int32_t* tok_of;      // [E][C] item (token * K + choice) of (expert, slot), valid for slot < count
  int32_t* local_rank;  // scratch [K*T]
  int32_t* block_hist;  // scratch [ceil(K*T/8)][E] (per gate tile of R >= 8 tokens, or per 1024 items)
  int32_t* tile_ties;   // scratch [ceil(T/8)]: ties per gate tile, summed by the slot scan
  int32_t* ties;        // [1]: tokens with gap < 1e-6
  // NEXT #4 gating variants
  int rts;              // random token-selection priority (R20)
  uint64_t seed;        //   its permutation key
  float aux_coef;       // > 0: auxiliary load-balancing loss (R21)
  float* aux_partial;   //   scratch [AUX_GRID][E] fp32 + [AUX_GRID][E] int32
  float* aux_out;       //   saved: f_e [E], then l_aux
};
cudaError_t route(const RouteArgs& a, cudaStream_t s);

// Slot-space layout [G_t][E][C_s][H]: slot c of expert e lives at slice c / C_s.
struct SlotSpace {
  int64_t C, Cs;  // capacity and slot-slice size
  int G_t, E, H;
  int K = 1;      // choices per token: per-token arrays are [T][K], tok_of holds token*K+choice
};

// F3: D[tt][e][cs] = x[tok_of[e][tt*Cs+cs]] (zeros for empty slots), for slices
// tt in [t_lo, t_hi). y_zero (or null): also zero the rows of tokens with slot[t] < 0.
cudaError_t dispatch(const void* x, const int32_t* tok_of, const int32_t* count,
                     const SlotSpace& ss, int t_lo, int t_hi, void* D, const int32_t* slot, int64_t T,
                     void* y_zero, cudaStream_t s);

// F11: y_t = bf16(sum over kept choices k of p_tk * O[row(t,k)]), 0 if all dropped.
cudaError_t combine(const void* O, const int32_t* expert, const int32_t* slot, const float* prob,
                    const SlotSpace& ss, int64_t T, void* y, cudaStream_t s);

// B1: dp_tk = <dy_t, O[row(t,k)]> (fp32, 0 if dropped), dO[row(t,k)] = bf16(p_tk dy_t) for
// kept choices whose slot lies in slices [t_lo, t_hi); empty slots in those slices -> 0.
cudaError_t combine_bwd(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                        const float* prob, const int32_t* count, const SlotSpace& ss, int64_t T,
                        int t_lo, int t_hi, float* dp, void* dO, cudaStream_t s);

// B10: dx_t = dS[row(t)] + sum_j dl_tj Wg[:, j] (kept), 0 (dropped);
// dl_tj = dp_t p_t (delta_{j,e*} - softmax(l_t)_j); dWg = sum_t x_t^T dl_t.
// (gate_bwd.cu) dl and the gathered slot-space rows grow [T][K] in a token-parallel pre-pass,
// dx by warp MMA; pack_scratch holds gate_bwd_pack_bytes(H, E).
// aux_f: f_e [E] of the aux loss (R21) and its coefficient, or null / 0.
cudaError_t gate_bwd(const void* x, const void* dS, const float* wg, const float* logits,
                     const int32_t* expert, const int32_t* slot, const float* prob,
                     const float* dp, const SlotSpace& ss, int64_t T, void* dx, float* dwg,
                     float* dl_scratch, int32_t* grow_scratch, float* dwg_partial, int nsplit, void* pack_scratch,
                     void* a_tok_scratch, int32_t* dwg_counters,
                     const float* aux_f, float aux_coef, cudaStream_t s);
int gate_bwd_splits(int64_t T);
// One-GPU top-1 (E <= 16) head of the backward in one launch: B1 (dp, dO incl. empty-slot
// zeros), dl, the EPI_SCATTER extension operands a_ext / b_ext, and zero dl / dx rows of
// dropped tokens (gate_bwd.cu).
cudaError_t combine_bwd_gate(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                             const float* prob, const float* logits, const int32_t* tok_of,
                             const int32_t* count, const float* wg, int64_t T, int H, int E, int64_t C,
                             void* dO, float* dl, void* a_ext, void* b_ext, void* dx, int32_t* dwg_cnt,
                             cudaStream_t s);
// dWg on the tensor cores from rows X [rows][H] and rows a_ext [rows][64] = [hi(dl) | lo(dl) | ...]
// (EP = 16 or 32 columns per block; one GPU: the dispatched rows and the K-extension rows,
// E <= 16; general B10 path: the token rows and [hi | lo](dl), E <= 32): one launch, split-K partials [<= max_split][H][E]
// summed in fixed order by the last CTA of each h tile; counters [ceil(H/128)] zeroed by
// combine_bwd_gate.
cudaError_t gate_dwg_tc(const void* X, const void* a_ext, int64_t rows, int H, int E, float* dwg, float* partial,
                        int max_split, int32_t* counters, cudaStream_t s);
// dWg = x^T dl (deterministic split-K), the tail of B10 on the fused path.
cudaError_t gate_dwg(const void* x, const float* dl, int64_t T, int H, int E, float* dwg, float* partial,
                     int nsplit, cudaStream_t s);
size_t gate_bwd_pack_bytes(int H, int E);

// (peer.cu) one piece of a peer-memory exchange: C_s x H bytes from src + src_off to
// window `win` of rank dst_rank at dst_off. kind: 0 local, 1 a2a (EP peer), 2 folded
// all-gather (TP peer) — used only by the byte ledger.
struct Piece {
  uint64_t src_off, dst_off;
  int32_t dst_rank, kind;
};
cudaError_t peer_exchange(const void* src, void* const* d_table, int nwin, int win,
                          const Piece* d_pieces, int npieces, size_t piece_bytes, cudaStream_t s);
// (peer.cu) fused TP reduction + return exchange for G_t > 1: reads the TP partials of
// window src_win (expert space) on every TP rank of this rank's group, writes the sums
// into window dst_win (slot space) of the source ranks.
struct ReduceReturn {
  void* const* table;  // device [world][nwin]
  int nwin, src_win, dst_win;
  int d, ep, t, Gt, Gep, El, E, H;
  int64_t Cs;
  int dtd;   // reduce only the rank's own slot slice
  int fold;  // and store it to every TP rank of the source (folded all-gather), else to the same t
  void* mc;  // MOE_F_NVLS direct: multicast mapping of dst_win over the own TP group (fold: rows
             // for the own EP group are stored once through it), or null
};
cudaError_t reduce_return(const ReduceReturn& rr, cudaStream_t s);
// (peer.cu) DTD all-gather in the TP group over NVLink SHARP multicast (MOE_F_NVLS):
// segments [base_off + i * stride, + seg_bytes), i < nseg, of window `win` of this rank are
// stored once through the group's multicast mapping `mc` (or, when null — emulated ranks —
// to each TP peer's window) at the same offsets. seg_bytes % 16 == 0.
struct TpAllGather {
  void* const* table;  // device [world][nwin]
  int nwin, win, rank, tp0, Gt;
  void* mc;            // multicast address of window `win`, or null
  uint64_t base_off, stride, seg_bytes;
  int nseg;
};
cudaError_t tp_allgather(const TpAllGather& ag, cudaStream_t s);
// (peer.cu) one-sided readiness flag: store `epoch` to flag (a peer's flag slot) after the
// stream's prior work; wait until *flag >= epoch (wrap-safe). Waits are bounded: after
// timeout_ns the kernel records a code in *err (host-mapped) and returns.
cudaError_t peer_signal(uint32_t* flag, uint32_t epoch, cudaStream_t s);
cudaError_t peer_wait(const uint32_t* flag, uint32_t epoch, int32_t* err, uint64_t timeout_ns, cudaStream_t s);
// Flag barrier over the peer windows (window `win` holds one uint32 slot per rank).
cudaError_t peer_barrier(void* const* d_table, int nwin, int win, int world, int rank,
                         uint32_t epoch, int32_t* err, uint64_t timeout_ns, cudaStream_t s);

// Destination of slot-space rows in the expert-space windows of the EP/TP peers
// (fused dispatch / combine-backward): slot (tt, e, cs) of this rank lands at
// [el][tt][ep][cs] of rank (d, e / E_l, t') for t' in {t} (vanilla) or all t' (DTD).
struct PeerDst {
  void* const* table;  // device [world][nwin]
  int nwin, win;
  int d, ep, t, Gt, Gep, El;
  int dtd;
  void* mc;  // MOE_F_NVLS direct: multicast mapping of `win` over this rank's TP group, or null;
             // with dtd, rows for the own EP group go once through it instead of G_t stores
};
// F3 + F4 (+F5): gather x rows of slices [t_lo, t_hi) straight into the peers' windows.
cudaError_t dispatch_peer(const void* x, const int32_t* tok_of, const int32_t* count,
                          const SlotSpace& ss, int t_lo, int t_hi, const PeerDst& pd,
                          cudaStream_t s);
// B1 + B2 (+B3): dp_t and dO rows (p_t dy_t, zeros for empty slots) straight into the peers' windows.
cudaError_t combine_bwd_peer(const void* dy, const void* O, const int32_t* expert,
                             const int32_t* slot, const float* prob, const int32_t* count,
                             const int32_t* tok_of, const SlotSpace& ss, int64_t T, int t_lo,
                             int t_hi, float* dp, const PeerDst& pd, cudaStream_t s);

// (optim.cu) the tiled optimizer step of include/moe_optim.h: binary32 scalars
// derived on the host in binary64 (reading R19).
struct AdamwScalars {
  float b1, b2, ob1, ob2, step, c2s, decay, eps;
};
cudaError_t adamw_fused(const void* grad, float* p, float* m, float* v, void* p16, int64_t n,
                        const AdamwScalars& s, cudaStream_t st);
cudaError_t adamw_tiled(const void* grad, float* p, float* m, float* v, void* p16, int64_t n,
                        const AdamwScalars& s, int64_t ts, float* temp, cudaStream_t st, int* launches);

// (permute.cu) G_t = 1 split exchange: rows of this rank's experts -> its own window
// (loc, expert space [E_l][G_ep][C][H], source block me), others -> stage (slot space
// [E][C][H]) for the copy-engine pieces of exchange_ce_dispatch.
struct SplitDst {
  void* loc;    // bf16
  void* stage;  // bf16
  int me, El, Gep;
};
cudaError_t dispatch_split(const void* x, const int32_t* tok_of, const int32_t* count,
                           const SlotSpace& ss, const SplitDst& sd, cudaStream_t s);
cudaError_t combine_bwd_split(const void* dy, const void* O, const int32_t* expert, const int32_t* slot,
                              const float* prob, const int32_t* count, const SlotSpace& ss, int64_t T,
                              float* dp, const SplitDst& sd, cudaStream_t s);

}  // namespace moe
