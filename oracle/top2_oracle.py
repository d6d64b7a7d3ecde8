"""Plain CPU oracle of top-2 gating (reading R22).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Shares no code with the
CUDA path. The top-1 oracle (moe_oracle.py) is untouched; this module reuses
only its bf16 decoding, GeLU and the R20/R21 helpers.

The paper cites the gate's lineage (GShard / Switch / DeepSpeed-MoE,
PAPER.md:96-97) without defining it. Reading R22 follows GShard's top-2:

  gate     l = x Wg; e1 = lowest argmax; e2 = lowest argmax over j != e1;
           s = softmax(l); S = s_e1 + s_e2; combine weights w1 = s_e1/S,
           w2 = s_e2/S (renormalised over the two choices);
           tie gap = min(l_e1 - l_e2, l_e2 - l_third) (either choice could flip).
  capacity C = ceil(cf * 2 T / E), >= 1, rounded up to a multiple of G_tensor.
  slots    all first choices in priority order, then all second choices in the
           same order, sharing each expert's C slots: the second choice of t
           gets load1_e + #{t' before t : e2(t') = e}; kept iff slot < C.
  forward  y_t = sum over kept choices k of w_tk * FFN_{e_k}(x_t).
  backward do_tk = w_tk dy_t, dw_tk = <dy_t, o_tk> (0 for a dropped choice);
           through the renormalisation: g1 = s2 (dw1 - dw2) / S^2,
           g2 = s1 (dw2 - dw1) / S^2; through the softmax:
           dl_tj = sum_k g_k s_{e_k} (delta_{j,e_k} - s_tj);
           dx_t = sum_k dh_tk W1_{e_k} + sum_j dl_tj Wg[:, j]; dWg = x^T dl.
  aux loss (R21) counts first choices only for f_e.
Everything in float64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .moe_oracle import aux_loss_dlogits, gelu_tanh, gelu_tanh_grad

__all__ = ["capacity_top2", "gate_top2", "assign_slots_top2", "Routing2", "route_top2", "layer_top2"]


def capacity_top2(tokens: int, experts: int, cf: float, g_tensor: int = 1) -> int:
    """C = ceil(cf * 2T / E), >= 1, rounded up to a multiple of G_tensor (R22, R2)."""
    c = max(int(math.ceil(cf * 2 * tokens / experts)), 1)
    return ((c + g_tensor - 1) // g_tensor) * g_tensor


def gate_top2(x: np.ndarray, wg: np.ndarray):
    """Returns (logits [T,E], experts [T,2], gap [T], s [T,E], w [T,2])."""
    logits = x @ wg
    T, E = logits.shape
    if E < 2:
        raise ValueError("top-2 needs E >= 2")
    ar = np.arange(T)
    e1 = np.argmax(logits, axis=1)
    masked = logits.copy()
    masked[ar, e1] = -np.inf
    e2 = np.argmax(masked, axis=1)
    l1, l2 = logits[ar, e1], logits[ar, e2]
    if E > 2:
        masked[ar, e2] = -np.inf
        l3 = masked.max(axis=1)
        gap = np.minimum(l1 - l2, l2 - l3)
    else:
        gap = l1 - l2
    z = np.exp(logits - l1[:, None])
    s = z / z.sum(axis=1, keepdims=True)
    experts = np.stack([e1, e2], axis=1).astype(np.int32)
    return logits, experts, gap, s, _weights(s, experts)


def _weights(s, experts):
    ar = np.arange(s.shape[0])
    s1, s2 = s[ar, experts[:, 0]], s[ar, experts[:, 1]]
    S = s1 + s2
    return np.stack([s1 / S, s2 / S], axis=1)


def assign_slots_top2(experts: np.ndarray, E: int, cap: int, order=None):
    """Returns (slot [T,2] int32 with -1 = dropped, count [E] kept, load [E] routed)."""
    T = experts.shape[0]
    slot = np.full((T, 2), -1, dtype=np.int32)
    seen = np.zeros(E, dtype=np.int64)
    seq = range(T) if order is None else [int(t) for t in order]
    for k in range(2):
        for t in seq:
            e = int(experts[t, k])
            if seen[e] < cap:
                slot[t, k] = seen[e]
            seen[e] += 1
    return slot, np.minimum(seen, cap).astype(np.int32), seen


@dataclass
class Routing2:
    logits: np.ndarray
    experts: np.ndarray  # [T,2]
    gap: np.ndarray
    s: np.ndarray
    w: np.ndarray        # [T,2]
    slot: np.ndarray     # [T,2]
    count: np.ndarray
    load: np.ndarray
    cap: int

    @property
    def kept(self) -> np.ndarray:  # [T,2]
        return self.slot >= 0


def route_top2(x, wg, cap, override=None, order=None) -> Routing2:
    """override: (idx, experts [len(idx),2]) — the tie protocol adopts the GPU's pair."""
    logits, experts, gap, s, w = gate_top2(x, wg)
    if override is not None:
        idx, ex = override
        experts = experts.copy()
        experts[np.asarray(idx, dtype=np.int64)] = np.asarray(ex, dtype=np.int32).reshape(-1, 2)
        w = _weights(s, experts)
    slot, count, load = assign_slots_top2(experts, wg.shape[1], cap, order)
    return Routing2(logits, experts, gap, s, w, slot, count, load, cap)


def _group(x, dy, wg, w1, w2, r: Routing2, aux_coef: float):
    T, H = x.shape
    E = wg.shape[1]
    y = np.zeros((T, H))
    dx = np.zeros((T, H))
    dw1 = np.zeros_like(w1)
    dw2 = np.zeros_like(w2)
    dwk = np.zeros((T, 2))   # dL/dw_tk
    for e in range(E):
        items = [(t, k) for k in range(2) for t in np.nonzero((r.experts[:, k] == e) & r.kept[:, k])[0]]
        if not items:
            continue
        ti = np.array([t for t, _ in items])
        ki = np.array([k for _, k in items])
        h = x[ti] @ w1[e].T
        a = gelu_tanh(h)
        o = a @ w2[e].T
        wt = r.w[ti, ki]
        np.add.at(y, ti, wt[:, None] * o)
        if dy is None:
            continue
        do = wt[:, None] * dy[ti]
        dwk[ti, ki] = np.sum(dy[ti] * o, axis=1)
        dh = (do @ w2[e]) * gelu_tanh_grad(h)
        np.add.at(dx, ti, dh @ w1[e])
        dw2[e] += do.T @ a
        dw1[e] += dh.T @ x[ti]
    if dy is None:
        return y, None
    ar = np.arange(T)
    s1 = r.s[ar, r.experts[:, 0]]
    s2 = r.s[ar, r.experts[:, 1]]
    S2 = (s1 + s2) ** 2
    g = np.stack([s2 * (dwk[:, 0] - dwk[:, 1]) / S2, s1 * (dwk[:, 1] - dwk[:, 0]) / S2], axis=1)
    dl = np.zeros((T, E))
    for k in range(2):
        sk = r.s[ar, r.experts[:, k]]
        onehot = np.zeros((T, E))
        onehot[ar, r.experts[:, k]] = 1.0
        dl += (g[:, k] * sk)[:, None] * (onehot - r.s)
    if aux_coef:
        dl += aux_loss_dlogits(r.experts[:, 0], r.s, aux_coef)
    dx += dl @ wg.T
    return y, (dx, x.T @ dl, dw1, dw2)


def layer_top2(xs, dys, wg, w1, w2, cf: float, g_tensor: int = 1, overrides=None, order=None,
               aux_coef: float = 0.0):
    """Top-2 layer over S token groups (as moe_oracle.layer). Returns dict with per-group
    'y', 'dx', 'dwg', 'routing', 'aux' and summed 'dw1', 'dw2'."""
    E = wg.shape[1]
    T = xs[0].shape[0]
    cap = capacity_top2(T, E, cf, g_tensor)
    out = {"y": [], "dx": [], "dwg": [], "routing": [], "aux": [], "cap": cap,
           "dw1": np.zeros_like(w1), "dw2": np.zeros_like(w2)}
    for s, x in enumerate(xs):
        r = route_top2(x, wg, cap, None if overrides is None else overrides[s], order)
        y, g = _group(x, None if dys is None else dys[s], wg, w1, w2, r, aux_coef)
        out["y"].append(y)
        out["routing"].append(r)
        f = np.bincount(r.experts[:, 0], minlength=E) / T
        out["aux"].append(float(aux_coef * E * np.sum(f * r.s.mean(axis=0))))
        if g is not None:
            out["dx"].append(g[0])
            out["dwg"].append(g[1])
            out["dw1"] += g[2]
            out["dw2"] += g[3]
    return out
