/*
 * moe.h — C ABI of the B200-native MoE layer (arXiv 2305.13525 hot path).
 *
 * The layer: top-1 gating with expert capacity, the dispatch permutation,
 * the expert-parallel all-to-all with Duplicate Token Dropping (DTD,
 * PAPER.md:1116-1163), the per-expert FFN (tensor-parallel over G_tensor,
 * PAPER.md:119-122) and the weighted combine. "Following previous work ...
 * every alternate layer has expert feedforward modules";
 * the gate itself is defined by BASELINE.json north_star and DESIGN.md
 * readings R1-R8 (the paper never specifies it).
 *
 * Process model: one process per GPU. Rank r = (d*G_expert + ep)*G_tensor + t
 * (R17): TP group = ranks sharing (d, ep); EP group = ranks sharing
 * (d, t). A TP group holds one token group of T tokens, replicated on its
 * G_tensor ranks (the Megatron all-reduce duplication).
 * Rank (d, ep, t) owns experts [ep*E_l, (ep+1)*E_l), E_l = E/G_expert, and
 * for each the F-slice [t*F/G_t, (t+1)*F/G_t): rows of W1 [F,H], columns of
 * W2 [H,F] (Megatron column/row split).
 *
 * World > 1 (default exchange): a communicator (moe_comm) owns peer-visible windows
 * (cudaMalloc, CUDA-IPC mapped on every rank of the box): a ring of ring_depth
 * forward windows (expert inputs X and combine sources O) plus the transient
 * backward / TP-partial windows and a flag page. One communicator serves every MoE
 * layer of the process (moe_comm_create + moe_create_on_comm), so window memory does
 * not grow with the number of layers; its size is moe_comm_plan_bytes. moe_create
 * builds a private communicator for a single layer. Calls of all contexts on one
 * communicator must be issued in the same order on every rank and stream-ordered
 * (one stream per rank).
 *
 * Conventions for every call:
 *  - Tensor pointers are caller-owned CUDA device pointers unless stated;
 *    the library never allocates, frees or retains them past the call.
 *    bf16 tensors are passed as void* (2-byte elements, row-major).
 *  - Work is enqueued asynchronously on the given stream (NCCL calls too);
 *    ordering is stream order. Outputs are overwritten, never accumulated.
 *  - Every call returns a moe_status; nothing throws or aborts across the
 *    ABI. Validation happens before anything is enqueued. A CUDA/NCCL
 *    failure poisons the ctx: later calls return MOE_ERR_STATE.
 *    moe_last_error_detail() gives a thread-local message for the last error.
 *  - A ctx is not thread-safe.
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOE_OK = 0,
  MOE_ERR_ARG = 1,         /* null pointer / out-of-range scalar                   */
  MOE_ERR_SHAPE = 2,       /* divisibility / size constraint violated              */
  MOE_ERR_ALIGN = 3,       /* pointer not 16-byte aligned (TMA / 16B vectors)      */
  MOE_ERR_STATE = 4,       /* wrong saved blob, poisoned ctx, missing comm         */
  MOE_ERR_CUDA = 5,        /* CUDA runtime / driver error                          */
  MOE_ERR_NCCL = 6,        /* NCCL error                                           */
  MOE_ERR_UNSUPPORTED = 7, /* valid request this build does not implement         */
  MOE_ERR_TIMEOUT = 8      /* a peer rank missed a window barrier / readiness signal
                              within moe_config.peer_timeout_ms (dead, absent or out
                              of step); the communicator and its contexts are broken */
} moe_status;

/* moe_config.flags */
#define MOE_F_STATS 1u            /* keep the per-collective byte ledger (moe_stats)        */
#define MOE_F_FORCED_ROUTING 2u   /* moe_forward takes forced_expert[T] instead of argmax   */
#define MOE_F_TIMING 4u           /* record CUDA events around every kernel class (moe_stats) */
#define MOE_F_NCCL_EXCHANGE 8u    /* EP exchange via NCCL send/recv + all-gather (baseline)
                                     instead of the peer-memory copy kernel (default)       */
#define MOE_F_CHECKPOINT 16u      /* activation checkpointing: the
                                     forward keeps the routing record and the outputs of its
                                     collectives (X, O: the CAC stash) but
                                     not G/A; moe_forward_replay re-materializes them before
                                     moe_backward                                           */
#define MOE_F_CAC 32u             /* with MOE_F_CHECKPOINT: the replay reuses the stash and
                                     issues no collectives (Communication-aware Activation
                                     Checkpointing); without it the replay
                                     re-runs the forward's collectives (plain checkpointing) */
#define MOE_F_NVLS 256u           /* DTD (g_tensor > 1, peer exchange) with the all-gathers on
                                     NVLink SHARP multicast: each
                                     rank sends its own slot slice to the same-t rank of the
                                     destination EP group (the a2a of 1/G_t of the tokens,
                                     PAPER.md:1153-1155) and then stores the slice it received
                                     once through its TP group's multicast mapping
                                     (multimem.st; the switch replicates it to every TP rank,
                                     PAPER.md:1155-1158) instead of writing G_t copies itself;
                                     same on the return and backward exchanges. Needs
                                     multicast-capable GPUs (MOE_ERR_UNSUPPORTED otherwise);
                                     emulated groups run the same data flow with unicast
                                     stores. Ignored without DTD in effect.                  */
/* Gating variants (the paper cites the gate's lineage,
 * PAPER.md:96-97, without defining it): */
#define MOE_F_RANDOM_PRIORITY 64u /* random token selection (R20): capacity slots
                                     are granted in a keyed pseudo-random order of the tokens
                                     (4-round Feistel permutation of [0, T), cycle-walked,
                                     key = moe_set_priority_seed) instead of token order     */
#define MOE_F_AUX_LOSS 128u       /* auxiliary load-balancing loss (R21):
                                     l_aux = aux_loss_coef * E * sum_e f_e P_e per token group,
                                     f_e = routed fraction, P_e = mean softmax probability;
                                     moe_forward computes it (moe_aux_loss reads it) and
                                     moe_backward adds d l_aux / d logits to the gate gradient
                                     of every token, dropped ones included                   */

/* Layer configuration. Identical on every rank of the job.
 * Constraints (checked, MOE_ERR_SHAPE otherwise):
 *   tokens >= 1; hidden % 64 == 0; experts in [1, 64];
 *   ffn % g_tensor == 0 and (ffn / g_tensor) % 64 == 0;
 *   experts % g_expert == 0; world == g_tensor * g_expert * G_data (G_data >= 1);
 *   capacity_factor > 0. */
typedef struct {
  int64_t tokens;          /* T: tokens per TP group, identical on its G_tensor ranks */
  int32_t hidden;          /* H                                                        */
  int32_t ffn;             /* F, unsharded                                             */
  int32_t experts;         /* E, global                                                */
  float capacity_factor;   /* cf                                                       */
  int32_t g_tensor;        /* G_tensor                                  */
  int32_t g_expert;        /* G_expert                                */
  int32_t dtd;             /* 0 = vanilla (AllReduce + full all-to-all), 1 = DTD       */
  uint32_t flags;          /* MOE_F_*                                                  */
  float aux_loss_coef;     /* MOE_F_AUX_LOSS coefficient (>= 0; ignored without the flag) */
  int32_t top_k;           /* experts per token: 0 or 1 = top-1 (R1), 2 = top-2 (DESIGN.md
                              R22: GShard renormalised weights, C = ceil(cf*2T/E), second
                              choices queue behind all first choices); top-2 needs
                              experts >= 2 and no MOE_F_FORCED_ROUTING. With top-2 the
                              per-token routing arrays become [T][2] (expert, slot, prob)  */
  int32_t ring_depth;      /* world > 1, peer exchange: forwards whose expert inputs X and
                              combine sources O stay in the communicator's windows until
                              their backward (0 = 2; at most 64). A saved blob stays valid
                              for moe_backward while fewer than ring_depth newer forwards
                              ran on the communicator (else MOE_ERR_STATE). Checkpointed
                              forwards (MOE_F_CHECKPOINT) take a slot while they run but
                              stash X/O in `saved`, so their backward needs none. Window
                              memory is moe_comm_plan_bytes.                              */
  int32_t peer_timeout_ms; /* deadline of every peer barrier / signal wait (0 = 60000);
                              a miss surfaces as MOE_ERR_TIMEOUT from the next call       */
} moe_config;

/* Per-rank derived layout (host-only; no GPU needed). */
typedef struct {
  int32_t world, rank;
  int32_t d, ep, t;        /* rank coordinates                                         */
  int32_t experts_local;   /* E_l = E / G_expert                                       */
  int32_t ffn_local;       /* F_l = F / G_tensor                                       */
  int64_t capacity;        /* C = ceil(cf*T/E) rounded up to a multiple of G_tensor, >= 1 (R2) */
  int64_t slot_slice;      /* C_s = C / G_tensor: one DTD slot slice                   */
  int64_t rows_per_expert; /* R = G_expert * C: GEMM rows of one local expert          */
  int32_t token_groups;    /* S = world / G_tensor                                     */
} moe_layout;

typedef struct moe_ctx moe_ctx;

/* Collective kinds in the ledger. */
enum { MOE_COLL_A2A = 0, MOE_COLL_ALLGATHER = 1, MOE_COLL_REDUCESCATTER = 2,
       MOE_COLL_ALLREDUCE = 3, MOE_COLL_KINDS = 4 };

/* One collective call of the forward+backward schedule (host-side plan).
 * wire_bytes: bytes this rank puts on NVLink for the call under the
 * lower-bound convention of PAPER.md:612-622 — all-to-all: bytes sent to
 * other ranks; all-gather / reduce-scatter: (s-1)/s x the full buffer;
 * all-reduce: 2(s-1)/s x the buffer (s = group size). */
typedef struct {
  int32_t kind;            /* MOE_COLL_*                                               */
  int32_t pass;            /* 0 = forward, 1 = backward, 2 = checkpoint replay          */
  int32_t step;            /* SURVEY §8(a) step id: 4,5,8,9,10 (F) / 2,3,7,8,9 (B)      */
  int32_t group_size;      /* s                                                        */
  int64_t buffer_bytes;    /* full buffer (a2a: send buffer incl. self chunk)          */
  int64_t wire_bytes;
} moe_collective;

/* Kernel classes of the ledger. */
enum { MOE_K_ROUTE = 0,       /* F1 gate + F2 slot scan                 */
       MOE_K_DISPATCH = 1,    /* F3                                     */
       MOE_K_GEMM = 2,        /* F6 F7 B4 B5 B6 (tcgen05 expert GEMMs)  */
       MOE_K_COMBINE = 3,     /* F11                                    */
       MOE_K_COMBINE_BWD = 4, /* B1                                     */
       MOE_K_GATE_BWD = 5,    /* B10                                    */
       MOE_K_COMM = 6,        /* NCCL collectives + self-chunk copies   */
       MOE_K_XFER = 7,        /* copy-engine exchange transfers (side stream, overlapped;
                                 timed, no kernels)                      */
       MOE_K_CLASSES = 8 };

typedef struct {
  int64_t calls[MOE_COLL_KINDS];
  int64_t wire_bytes[MOE_COLL_KINDS];
  int64_t forward_calls, backward_calls;
  int64_t dropped_tokens;  /* last forward: (token, choice) pairs beyond capacity (this group) */
  int64_t tie_tokens;      /* last forward: top-2 gap < 1e-6 (logged ties)            */
  int32_t nccl_async_error;/* ncclCommGetAsyncError of the last check (0 = none)      */
  int64_t kernel_launches[MOE_K_CLASSES]; /* CUDA kernels this library launched, per class */
  double kernel_ms[MOE_K_CLASSES];        /* MOE_F_TIMING: summed CUDA-event time per class */
  int64_t replay_calls;                   /* collectives issued by moe_forward_replay       */
} moe_stats;

/* ---------------- host-only planning (no GPU, no ctx) ---------------- */

/* Validates cfg for (world, rank) and fills the derived layout. */
moe_status moe_plan_layout(const moe_config* cfg, int world, int rank, moe_layout* out);

/* Sizes of the caller-allocated buffers: saved (one forward's stash for its
 * backward: routing record, expert inputs X, Hpre, A = gelu(Hpre), combine
 * source O) and scratch (transient; may be shared by consecutive calls on one
 * stream). Both must be 256-byte aligned device memory. The saved blob keeps
 * G = gelu'(Hpre) rather than Hpre itself (the backward only needs gelu'). */
moe_status moe_plan_bytes(const moe_config* cfg, int world, int rank,
                          size_t* saved_bytes, size_t* scratch_bytes);

/* The collective schedule of one forward+backward on this rank, in issue
 * order (the ledger moe_forward/moe_backward actually follow). If out is
 * NULL or cap is too small only *n is written. */
moe_status moe_plan_collectives(const moe_config* cfg, int world, int rank,
                                moe_collective* out, int cap, int* n);

/* ---------------- context ---------------- */

/* Rank 0 creates the NCCL unique id; the caller broadcasts the 128 bytes
 * (e.g. with torch.distributed) before moe_create. */
moe_status moe_get_unique_id(uint8_t uid[128]);

/* Collective over the world when world > 1 (ncclCommInitRank + ncclCommSplit
 * into the TP and EP communicators); uid is ignored when world == 1. The CUDA
 * device must already be current. scratch/scratch_bytes: caller-owned device
 * buffer of at least moe_plan_bytes' scratch size, used by every call on this
 * ctx. */
moe_status moe_create(const moe_config* cfg, const uint8_t uid[128], int world, int rank,
                      void* scratch, size_t scratch_bytes, moe_ctx** out);

/* ---------------- communicator shared by the layers of a process ----------------
 *
 * moe_comm_plan_bytes: device bytes moe_comm_create allocates on this rank for the
 * layers `cfgs[0..n)` (windows sized for the largest; all layers need the same
 * g_tensor / g_expert; ring depth and deadline = the largest requested). 0 when no
 * layer uses the peer exchange (world == 1, or MOE_F_NCCL_EXCHANGE only). NCCL's own
 * buffers (NCCL-exchange layers only) are not included. Host-only. */
typedef struct moe_comm moe_comm;
moe_status moe_comm_plan_bytes(const moe_config* cfgs, int n, int world, int rank, size_t* device_bytes);

/* Collective over the world (world > 1): peer windows exchanged once over a temporary
 * NCCL communicator (kept only when a layer uses MOE_F_NCCL_EXCHANGE). */
moe_status moe_comm_create(const moe_config* cfgs, int n, const uint8_t uid[128], int world, int rank,
                           moe_comm** out);
/* Destroy after every context created on it (MOE_ERR_STATE otherwise). */
moe_status moe_comm_destroy(moe_comm* comm);

/* A layer context on a shared communicator (cfg must be one of the configs the
 * communicator was planned for, or fit in its windows). */
moe_status moe_create_on_comm(const moe_config* cfg, moe_comm* comm, void* scratch, size_t scratch_bytes,
                              moe_ctx** out);

/* ---------------- emulated ranks (one process, one device) ----------------
 * Runs the world > 1 path of every rank of a (g_tensor, g_expert) layout on ONE GPU:
 * each rank is a host thread with its own stream and its own moe_comm / moe_ctx made by
 * moe_comm_create_emulated on the group (blocks until all `world` ranks joined). The
 * ranks' windows are ordinary allocations on the group's device; every exchange,
 * TP-reduction and combine kernel is the same as with one process per GPU, only the
 * publication differs: a barrier is a host barrier plus cudaStreamWaitEvent on every
 * rank's event, a readiness signal is an event (no kernel waits on another kernel).
 * The NCCL exchange (MOE_F_NCCL_EXCHANGE) cannot be emulated (MOE_ERR_UNSUPPORTED).
 * Create the group with the device current; destroy it after every rank's comm. */
typedef struct moe_emu_group moe_emu_group;
moe_status moe_emu_group_create(int world, moe_emu_group** out);
moe_status moe_emu_group_destroy(moe_emu_group* group);
moe_status moe_comm_create_emulated(const moe_config* cfgs, int n, moe_emu_group* group, int rank,
                                    moe_comm** out);

/* Forward.
 *   x      bf16 [T, H]            tokens of this rank's TP group
 *   wg     fp32 [H, E]            gate weight (replicated)
 *   w1     bf16 [E_l, F_l, H]     this rank's W1 shards
 *   w2     bf16 [E_l, H, F_l]     this rank's W2 shards
 *   y      bf16 [T, H]            output: p_t * FFN_{e_t}(x_t), 0 for dropped tokens
 *   saved  device blob of moe_plan_bytes' saved size (written)
 *   forced_expert  int32 [T] or NULL; required iff MOE_F_FORCED_ROUTING. */
moe_status moe_forward(moe_ctx* ctx, const void* x, const float* wg, const void* w1,
                       const void* w2, void* y, void* saved, const int32_t* forced_expert,
                       void* stream);

/* Backward. dy bf16 [T, H]; saved from this ctx's
 * forward on the same x/wg/w1/w2. Outputs (overwritten):
 *   dx  bf16 [T, H]; dwg fp32 [H, E] (this token group's gradient);
 *   dw1 bf16 [E_l, F_l, H]; dw2 bf16 [E_l, H, F_l] (summed over every token
 *   routed to the shard within its EP group; no data-parallel reduction). */
moe_status moe_backward(moe_ctx* ctx, const void* dy, const void* saved, const void* x,
                        const float* wg, const void* w1, const void* w2, void* dx,
                        float* dwg, void* dw1, void* dw2, void* stream);

/* Checkpoint replay (MOE_F_CHECKPOINT only): re-materializes G = gelu'(Hpre)
 * and A = gelu(Hpre) of a checkpointed forward into the ctx scratch, ahead of
 * moe_backward on the same saved blob. With MOE_F_CAC the replay runs GEMM1 on
 * the stashed expert inputs X and issues no collective; otherwise it re-runs the
 * forward (gate, dispatch, exchanges, GEMMs, TP reduction) including every
 * collective, as plain activation checkpointing does. Arguments as moe_forward.
 * The scratch holds one replay at a time: replay, then backward, per layer. */
moe_status moe_forward_replay(moe_ctx* ctx, const void* saved, const void* x, const float* wg,
                              const void* w1, const void* w2, void* stream);

/* Copies the routing record of a saved blob (device -> device, async).
 * expert/slot int32 [T][K] (slot -1 = dropped), prob fp32 [T][K] (the combine
 * weights), gap fp32 [T] (top-2: min of the top-1/2 and top-2/3 logit gaps),
 * count int32 [E] (kept per expert, <= C); K = 1 or top_k. Any output may be NULL. */
moe_status moe_routing(moe_ctx* ctx, const void* saved, int32_t* expert, int32_t* slot,
                       float* prob, float* gap, int32_t* count, void* stream);

/* MOE_F_AUX_LOSS: copies this forward's l_aux (fp32, device pointer, async).
 * MOE_ERR_STATE without the flag or for a saved blob no forward wrote. */
moe_status moe_aux_loss(moe_ctx* ctx, const void* saved, float* aux, void* stream);

/* MOE_F_RANDOM_PRIORITY: the key of the priority permutation used by every later
 * moe_forward on this ctx (default 0). A training loop sets a new key per step;
 * the same key gives the same slots (the replay and backward use the saved ones). */
moe_status moe_set_priority_seed(moe_ctx* ctx, uint64_t seed);

/* Ledger + last-forward routing counters + per-class kernel launches/times;
 * synchronizes the ctx's last stream. */
moe_status moe_stats_get(moe_ctx* ctx, moe_stats* out);
moe_status moe_stats_reset(moe_ctx* ctx);
/* MOE_F_TIMING's per-class CUDA events on (on != 0) or off for the following calls of
 * this ctx (the events sit between kernel launches, so a throughput measurement turns
 * them off and a per-class breakdown turns them on). Without MOE_F_TIMING: MOE_ERR_STATE. */
moe_status moe_set_timing(moe_ctx* ctx, int on);

moe_status moe_destroy(moe_ctx* ctx);

const char* moe_status_string(moe_status s);
const char* moe_last_error_detail(void);

/* ---------------- diagnostics: the expert GEMM on its own ----------------
 * D[b] = epilogue(A[b] . B[b]^T) for b < batch, bf16 in, fp32 accumulate in
 * TMEM (tcgen05), bf16 out. Used by the tests and the GEMM micro-benchmark.
 *   A: a_mn == 0 -> [batch][M][K] (K-major);  a_mn == 1 -> [batch][K][M]
 *   B: b_mn == 0 -> [batch][N][K] (K-major);  b_mn == 1 -> [batch][K][N]
 *   D: [batch][M][N].  M, K >= 1; N % 64 == 0; M, K, N multiples of 8.
 *   epilogue 0: D = bf16(acc)
 *   epilogue 1: D = bf16(gelu_tanh'(acc)), aux = bf16(gelu_tanh(acc)) [batch][M][N]
 *               (the forward FFN GEMM: A for the second GEMM, G = gelu'(Hpre) for B4)
 *   epilogue 2: D = bf16(acc * aux), aux = G bf16 [batch][M][N] (read) (dGeLU)
 *   impl 0: tcgen05 CTA-pair kernel (cta_group::2, the product path);
 *   impl 1: plain SIMT reference kernel (bring-up cross-check only; never used
 *   by moe_forward/backward); anything else: MOE_ERR_UNSUPPORTED. */
moe_status moe_gemm_bf16(int batch, int M, int N, int K, const void* A, int a_mn,
                         const void* B, int b_mn, void* D, int epilogue, void* aux,
                         int impl, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
