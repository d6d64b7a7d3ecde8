"""Plain CPU oracle of the paper's tiled optimizer step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and
bench.py's CPU legs, never by the product path. Shares no code with
paper_2305_13525_b200/csrc.

What the paper says:
  "An intermediate step in the optimizer phase in mixed precision training is
  the up-casting of 16-bit gradients to 32-bit gradients before the optimizer
  updates the weights. This requires the creation of a temporary buffer to
  store the 32-bit gradients" — the untiled step;
  "partitioning these parameters into ``tiles'' of a predefined size and
  iteratively processing these tiles ... temporary 32-bit gradients are only
  produced for parameters belonging to a given tile. The temporary memory used
  to store these gradients can in fact be reused across tiles. For a tile size
  ts, we now only need 4 x ts bytes"; "we fix the tile size to
  1.8 million parameters" — the tiled step.

The update rule is not written in the paper (the companion runs in PAPER.md
use "mixed precision training ... and the AdamW optimizer");
reading R19 fixes decoupled-weight-decay Adam (Loshchilov &
Hutter, Alg. 2) in the PyTorch operation order, every
operation a single IEEE-754 binary32 operation (numpy float32 scalars and
arrays round every +, -, *, /, sqrt correctly), no fused multiply-add:

  host (binary64):  c1 = 1 - b1**t,  c2 = 1 - b2**t
                    step = f32(lr / c1),  c2s = f32(sqrt(c2)),
                    decay = f32(1 - lr * wd),  ob1 = f32(1 - b1),  ob2 = f32(1 - b2)
  per element:      g  = f32(grad16)                       (exact upcast)
                    m' = b1 * m + ob1 * g
                    v' = b2 * v + ob2 * (g * g)
                    p1 = p * decay
                    d  = sqrt(v') / c2s + eps
                    p' = p1 - step * (m' / d)
                    p16 = bf16_rn(p')                      (the 16-bit model copy)

Because every element's update reads only that element, tiling cannot
change a bit (the paper's premise); the oracle nevertheless executes the
tiled step literally (one reused ts-element float32 buffer, tiles in
ascending order) and reports its peak transient bytes, so tests can check the
"4 x ts" law against the untiled "4 x n".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["AdamW", "host_scalars", "tile_plan", "adamw_untiled", "adamw_tiled", "bf16_round_bits",
           "TILE_PARAMS_PAPER"]

# "we fix the tile size to 1.8 million parameters"
TILE_PARAMS_PAPER = 1_800_000


@dataclass(frozen=True)
class AdamW:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    step: int = 1  # t >= 1: the step being taken


def host_scalars(h: AdamW):
    """The per-step scalars, computed in binary64 and rounded once to binary32."""
    if h.step < 1:
        raise ValueError("step must be >= 1")
    c1 = 1.0 - h.beta1 ** h.step
    c2 = 1.0 - h.beta2 ** h.step
    f = np.float32
    return {"b1": f(h.beta1), "b2": f(h.beta2), "ob1": f(1.0 - h.beta1), "ob2": f(1.0 - h.beta2),
            "step": f(h.lr / c1), "c2s": f(math.sqrt(c2)), "decay": f(1.0 - h.lr * h.weight_decay),
            "eps": f(h.eps)}


def bf16_round_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even (NaN not expected here)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def _upcast(grad_bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float32 (exact)."""
    return (np.asarray(grad_bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _update(g, p, m, v, s):
    """One element-wise AdamW update on float32 arrays, in the order of the module docstring."""
    m2 = s["b1"] * m + s["ob1"] * g
    v2 = s["b2"] * v + s["ob2"] * (g * g)
    p1 = p * s["decay"]
    d = np.sqrt(v2) / s["c2s"] + s["eps"]
    p2 = p1 - s["step"] * (m2 / d)
    return p2.astype(np.float32), m2.astype(np.float32), v2.astype(np.float32)


def tile_plan(n: int, ts: int):
    """[start, end) ranges of at most ts parameters covering [0, n), ascending."""
    if ts < 1:
        raise ValueError("tile size must be >= 1")
    return [(a, min(a + ts, n)) for a in range(0, n, ts)]


def adamw_untiled(grad_bits, master, exp_avg, exp_avg_sq, h: AdamW):
    """The baseline the paper fixes: one float32 buffer for all n gradients.
    Returns (master', exp_avg', exp_avg_sq', param_bf16_bits, peak_transient_bytes)."""
    s = host_scalars(h)
    g32 = _upcast(grad_bits)                    # the full-length temporary
    p, m, v = _update(g32, np.asarray(master, np.float32), np.asarray(exp_avg, np.float32),
                      np.asarray(exp_avg_sq, np.float32), s)
    return p, m, v, bf16_round_bits(p), 4 * len(g32)


def adamw_tiled(grad_bits, master, exp_avg, exp_avg_sq, h: AdamW, ts: int):
    """The paper's tiled step: one reused ts-element float32 buffer."""
    s = host_scalars(h)
    n = len(grad_bits)
    p = np.array(master, dtype=np.float32, copy=True)
    m = np.array(exp_avg, dtype=np.float32, copy=True)
    v = np.array(exp_avg_sq, dtype=np.float32, copy=True)
    buf = np.empty(min(ts, n), dtype=np.float32)  # allocated once, reused by every tile
    for a, b in tile_plan(n, ts):
        k = b - a
        buf[:k] = _upcast(grad_bits[a:b])
        p[a:b], m[a:b], v[a:b] = _update(buf[:k], p[a:b], m[a:b], v[a:b], s)
    return p, m, v, bf16_round_bits(p), 4 * len(buf)
