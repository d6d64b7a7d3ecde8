/* moe_optim.h — the paper's tiled optimizer step for the expert parameters
 * (SURVEY.md §8(f) NEXT #3), exported by the same libmoe.so as moe.h.
 *
 * mixed-precision training up-casts the 16-bit gradients to a
 * temporary 32-bit buffer before the optimizer updates the weights; for the
 * expert parameter group (reduced data parallelism) that buffer
 * is the step's memory spike. PAPER.md:70-81: partition the parameters into
 * tiles of ts parameters and process them one after another, reusing one
 * 4*ts-byte buffer; ts = 1.8 M (MOE_TILE_PARAMS_PAPER).
 *
 * Update rule (reading R19; the paper names AdamW):
 * decoupled-weight-decay Adam, every operation one IEEE binary32 operation in
 * this order (no fused multiply-add), with the per-step scalars computed in
 * binary64 on the host and rounded once to binary32:
 *   c1 = 1 - beta1^t, c2 = 1 - beta2^t, step = lr / c1, c2s = sqrt(c2),
 *   decay = 1 - lr * weight_decay, ob1 = 1 - beta1, ob2 = 1 - beta2;
 *   g = f32(grad16); m = beta1*m + ob1*g; v = beta2*v + ob2*(g*g);
 *   p = p*decay - step*(m / (sqrt(v)/c2s + eps)); param16 = bf16_rn(p).
 * The result is bit-identical for every tile size (the rule is element-wise)
 * and bit-identical to oracle/optim_oracle.py.
 */
#ifndef MOE_OPTIM_H
#define MOE_OPTIM_H

#include <stddef.h>
#include <stdint.h>

#include "moe.h"

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_TILE_PARAMS_PAPER 1800000

typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
  int64_t step; /* t >= 1: the step being taken (bias correction) */
} moe_adamw_hparams;

/* Tile plan of the tiled step: n_tiles = ceil(n / tile_params) and the bytes of
 * the reused fp32 gradient buffer, 4 * min(tile_params, n).
 * tile_params = 0 asks for the fused step (no buffer: n_tiles = 1, temp 0).
 * Errors: MOE_ERR_ARG for n < 0, tile_params < 0 or null outputs. */
moe_status moe_adamw_plan(int64_t n, int64_t tile_params, int64_t* n_tiles, size_t* temp_bytes);

/* One optimizer step over n parameters, enqueued on `stream`; all pointers are
 * caller-owned device memory, 16-byte aligned:
 *   grad        bf16 [n]  16-bit gradients (read)
 *   master      f32  [n]  32-bit master weights (updated in place)
 *   exp_avg     f32  [n]  first moment (updated in place)
 *   exp_avg_sq  f32  [n]  second moment (updated in place)
 *   param       bf16 [n]  16-bit model copy written from the new master (nullable)
 * tile_params > 0: the paper's tiled step — for each tile (ascending), one kernel
 *   up-casts its gradients into `temp` (>= moe_adamw_plan's temp_bytes) and one
 *   kernel applies the update from `temp` (2 launches per tile).
 * tile_params = 0: the B200 step — one streaming kernel up-casts in registers
 *   (no temporary at all); `temp` must be NULL.
 * Errors (nothing enqueued): MOE_ERR_ARG (null pointer, n < 0, step < 1, temp
 * missing / unexpected), MOE_ERR_ALIGN (pointer not 16-byte aligned),
 * MOE_ERR_CUDA (launch failure). */
moe_status moe_adamw_step(const void* grad, float* master, float* exp_avg, float* exp_avg_sq,
                          void* param, int64_t n, const moe_adamw_hparams* h,
                          int64_t tile_params, float* temp, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_OPTIM_H */
