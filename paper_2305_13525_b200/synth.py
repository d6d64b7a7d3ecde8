"""Seeded synthetic inputs for the MoE layer hot path.

This module is shared by the tests, the bench and smoke(): it produces the
*inputs* only (tokens, gate weights, expert weights, upstream gradients,
forced routings) and holds none of the method's arithmetic. Both the CUDA path
and the CPU oracle (oracle/) are fed from here; neither imports the other.

Recipe:
  x  ~ N(0, 1)            -> bf16   [T, H]      seed BASE + group
  Wg ~ N(0, 1/H)          -> fp32   [H, E]      seed BASE + 1000   (logits ~ N(0,1))
  W1 ~ N(0, 1/H)          -> bf16   [E, F, H]   seed BASE + 2000 + e
  W2 ~ N(0, 1/F)          -> bf16   [E, H, F]   seed BASE + 2000 + e (second draw)
  dy ~ N(0, 1)            -> bf16   [T, H]      seed BASE + 3000 + group
"skewed" multiplies Wg[:, 0] by 1.5 so expert 0 is oversubscribed and drops.
T = 16384 = 8 sequences x 2048 tokens (GPT-style sequence length 2048,
PAPER.md:753, 831). bf16 values are carried as uint16 bit patterns.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

BASE_SEED = 230513525


def f32_to_bf16_bits(a) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round-to-nearest-even (no NaNs expected)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b) -> np.ndarray:
    """bf16 bit pattern -> fp32, exact."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


@dataclass(frozen=True)
class LayerShape:
    """One MoE-layer workload (BASELINE.json configs)."""
    name: str
    tokens: int          # T: tokens per tensor-parallel group
    hidden: int          # H
    ffn: int             # F (unsharded)
    experts: int         # E (global)
    cf: float = 1.0      # capacity factor
    g_tensor: int = 1    # G_tensor
    g_expert: int = 1    # G_expert

    @property
    def world(self) -> int:
        return self.g_tensor * self.g_expert

    @property
    def groups(self) -> int:
        """S: number of distinct token groups (= world / G_tensor, G^e_data = 1)."""
        return self.g_expert

    def with_(self, **kw) -> "LayerShape":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: the oracle finishes in seconds.
    "tiny": LayerShape("tiny", 256, 64, 256, 4),
    # configs[1]: the bench workload at N=1.
    "1.3b": LayerShape("1.3b", 16384, 2048, 8192, 16),
    # configs[2]: expert parallel over 8 GPUs.
    "2.7b-ep8": LayerShape("2.7b-ep8", 16384, 2560, 10240, 32, g_expert=8),
    # configs[3]: G_tensor = 2, G_expert = 4, DTD vs vanilla.
    "6.7b-tp2ep4": LayerShape("6.7b-tp2ep4", 16384, 4096, 16384, 16, g_tensor=2, g_expert=4),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def make_x(shape: LayerShape, group: int = 0, tokens: int | None = None) -> np.ndarray:
    T = shape.tokens if tokens is None else tokens
    g = _rng(BASE_SEED + group)
    return f32_to_bf16_bits(g.standard_normal((T, shape.hidden), dtype=np.float32))


def make_wg(shape: LayerShape, skew: float = 1.0) -> np.ndarray:
    g = _rng(BASE_SEED + 1000)
    wg = g.standard_normal((shape.hidden, shape.experts), dtype=np.float32)
    wg *= np.float32(1.0 / math.sqrt(shape.hidden))
    if skew != 1.0:
        wg[:, 0] *= np.float32(skew)
    return np.ascontiguousarray(wg, dtype=np.float32)


def make_expert(shape: LayerShape, e: int) -> tuple[np.ndarray, np.ndarray]:
    """(W1_e [F, H], W2_e [H, F]) as bf16 bits for global expert e."""
    g = _rng(BASE_SEED + 2000 + e)
    w1 = g.standard_normal((shape.ffn, shape.hidden), dtype=np.float32)
    w1 *= np.float32(1.0 / math.sqrt(shape.hidden))
    w2 = g.standard_normal((shape.hidden, shape.ffn), dtype=np.float32)
    w2 *= np.float32(1.0 / math.sqrt(shape.ffn))
    return f32_to_bf16_bits(w1), f32_to_bf16_bits(w2)


def make_experts(shape: LayerShape, experts: range | None = None):
    """Stacked (W1 [E', F, H], W2 [E', H, F]) bf16 bits for the listed experts."""
    ids = range(shape.experts) if experts is None else experts
    pairs = [make_expert(shape, e) for e in ids]
    return (np.stack([p[0] for p in pairs]), np.stack([p[1] for p in pairs]))


def make_dy(shape: LayerShape, group: int = 0, tokens: int | None = None) -> np.ndarray:
    T = shape.tokens if tokens is None else tokens
    g = _rng(BASE_SEED + 3000 + group)
    return f32_to_bf16_bits(g.standard_normal((T, shape.hidden), dtype=np.float32))


def forced_routing(mode: str, tokens: int, experts: int, seed: int = 0) -> np.ndarray:
    """Forced expert ids (int32 [T]) for the routing stress modes.

    round_robin: token t -> t mod E (no drops at cf >= 1).
    all_to_one : every token -> expert 0 (maximum drops).
    random     : uniform random experts (seeded).
    """
    if mode == "round_robin":
        return (np.arange(tokens) % experts).astype(np.int32)
    if mode == "all_to_one":
        return np.zeros(tokens, dtype=np.int32)
    if mode == "random":
        return _rng(BASE_SEED + 4000 + seed).integers(0, experts, tokens).astype(np.int32)
    raise ValueError(mode)


def shard_experts(w1: np.ndarray, w2: np.ndarray, shape: LayerShape, ep: int, t: int):
    """Rank (ep, t)'s shards: experts [ep*E_l, (ep+1)*E_l), W1 rows and W2
    columns [t*F/G_t, (t+1)*F/G_t) (Megatron column/row split)."""
    El = shape.experts // shape.g_expert
    Fl = shape.ffn // shape.g_tensor
    es = slice(ep * El, (ep + 1) * El)
    fs = slice(t * Fl, (t + 1) * Fl)
    return (np.ascontiguousarray(w1[es, fs, :]), np.ascontiguousarray(w2[es, :, fs]))
