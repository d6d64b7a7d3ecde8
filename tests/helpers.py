"""Shared test helpers: seeded inputs -> torch/oracle, parity metrics, tie protocol."""
from __future__ import annotations

import numpy as np
import torch

from oracle import moe_oracle as O
from paper_2305_13525_b200 import synth

REL_L2_BAR = 1e-2  # BASELINE.json north_star: relative L2 <= 1e-2 (bf16, fp32 accumulate)


def bf16_tensor(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


def tensor_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def rel_l2(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nr = np.linalg.norm(ref)
    if nr == 0:
        return 0.0 if np.linalg.norm(got) == 0 else np.inf
    return float(np.linalg.norm(got - ref) / nr)


class Inputs:
    """Seeded inputs of one workload (all token groups), as bf16 bits + fp32 Wg."""

    def __init__(self, shape: synth.LayerShape, tokens: int | None = None, skew: float = 1.0):
        self.shape = shape
        self.T = shape.tokens if tokens is None else tokens
        S = shape.groups
        self.x = [synth.make_x(shape, s, self.T) for s in range(S)]
        self.dy = [synth.make_dy(shape, s, self.T) for s in range(S)]
        self.wg = synth.make_wg(shape, skew)
        self.w1, self.w2 = synth.make_experts(shape)

    def oracle_arrays(self):
        return ([O.decode_bf16(a) for a in self.x], [O.decode_bf16(a) for a in self.dy],
                self.wg.astype(np.float64), O.decode_bf16(self.w1), O.decode_bf16(self.w2))


def routing_protocol(gpu_expert, gpu_gap, r: O.Routing):
    """SURVEY §8(c) comparison step 2: argmax must match outside the tie set
    (top-2 gap < 1e-6 on either side); returns (tie_idx, override experts)."""
    ge = np.asarray(gpu_expert)
    tie = (r.gap < O.TIE_GAP) | (np.asarray(gpu_gap) < O.TIE_GAP)
    bad = np.nonzero((ge != r.expert) & ~tie)[0]
    assert bad.size == 0, f"routing mismatch outside tie set at tokens {bad[:10]}"
    idx = np.nonzero(tie)[0]
    return idx, ge[idx]


ROW_REL_BAR = 5e-2  # per-row bound beside the global one: a single corrupted row cannot hide
ROW_FLOOR = 0.1    # row denominators never below 10% of the tensor's RMS row norm


def row_errors(got, ref, axis_rows: int = -1):
    """Per-row relative L2 of got vs ref (rows = all but the last axis). Rows whose
    reference is exactly zero (dropped tokens, experts with no tokens) must be exactly
    zero on the GPU too; returns (max rel over nonzero rows, #zero rows violated).

    The denominator of a row is max(|ref_row|, ROW_FLOOR * RMS of the nonzero row norms)
    (DESIGN.md §5): a row whose true norm is a small fraction of the typical row — e.g. a
    dW1 row of a single token where gelu'(Hpre_f) ~ 0, so the bf16 rounding of Hpre is a
    large relative error of that row — is judged against the row scale of its tensor; a
    corrupted row (error of the order of a typical row) still fails."""
    g = np.asarray(got, dtype=np.float64).reshape(-1, np.asarray(got).shape[-1])
    r = np.asarray(ref, dtype=np.float64).reshape(-1, np.asarray(ref).shape[-1])
    nr = np.linalg.norm(r, axis=1)
    nd = np.linalg.norm(g - r, axis=1)
    nz = nr > 0
    floor = ROW_FLOOR * float(np.sqrt(np.mean(nr[nz] ** 2))) if nz.any() else 0.0
    worst = float((nd[nz] / np.maximum(nr[nz], floor)).max()) if nz.any() else 0.0
    bad_zero = int(np.count_nonzero(nd[~nz] > 0))
    return worst, bad_zero


def parity_failures(name: str, got, ref, rows: bool = True) -> list[str]:
    """Global rel L2 <= 1e-2 (BASELINE.json) and, per row, <= 5e-2 with exact zeros."""
    out = []
    e = rel_l2(got, ref)
    if not e <= REL_L2_BAR:
        out.append(f"{name}: rel L2 {e:.3e} > {REL_L2_BAR}")
    if rows and np.asarray(ref).ndim >= 2:
        worst, bad_zero = row_errors(got, ref)
        if not worst <= ROW_REL_BAR:
            out.append(f"{name}: worst row rel L2 {worst:.3e} > {ROW_REL_BAR}")
        if bad_zero:
            out.append(f"{name}: {bad_zero} rows nonzero where the oracle is exactly zero")
    return out


class LazyExperts:
    """Expert weights decoded to float64 one expert at a time (full-size shapes do not fit
    as a float64 [E, F, H] array); indexable like the stacked array: w[e] -> [F, H]."""

    def __init__(self, bits):
        self.bits = bits
        self._e, self._v = None, None

    def __getitem__(self, e):
        e = int(e)
        if e != self._e:
            self._e, self._v = e, O.decode_bf16(self.bits[e])
        return self._v


def stratified_tokens(r: "O.Routing", src_block: int, tile: int = 256, seed: int = 0, extra: int = 4):
    """One kept token per (expert, `tile`-row M-tile) of the expert GEMMs — a token of
    source block s with slot c is row s*C + c of its expert's [G_ep*C] rows — plus a few
    dropped tokens and the first / last token. Covers every M-tile of every expert."""
    rng = np.random.default_rng(seed)
    picks = [0, len(r.expert) - 1]
    for e in range(len(r.count)):
        kept = np.nonzero((r.expert == e) & r.kept)[0]
        if kept.size == 0:
            continue
        tiles = (src_block * r.cap + r.slot[kept]) // tile
        for tl in np.unique(tiles):
            picks.append(int(rng.choice(kept[tiles == tl])))
    dropped = np.nonzero(~r.kept)[0]
    if dropped.size:
        picks += [int(t) for t in rng.choice(dropped, min(extra, dropped.size), replace=False)]
    return np.array(sorted(set(picks)), dtype=np.int64)


def stratified_f(F_local: int, tile: int = 256, seed: int = 0):
    """One index per `tile`-wide block of [0, F_local): covers every dW1 M-tile (rows f)
    and every dW2 N-tile (columns f) of the weight-gradient GEMMs."""
    rng = np.random.default_rng(seed)
    return np.array([min(b + int(rng.integers(tile)), F_local - 1) for b in range(0, F_local, tile)])
