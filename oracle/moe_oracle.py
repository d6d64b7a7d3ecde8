"""Plain, slow, obviously-correct CPU oracle of the MoE layer forward/backward.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs, never by the
product path. Shares no code with paper_2305_13525_b200/csrc.

What it computes (readings R1-R17 are listed in DESIGN.md):
the MoE layer of arXiv 2305.13525 — "every alternate layer has expert
feedforward modules" — with top-1 gating and expert capacity
as named by BASELINE.json north_star (the paper never defines the gate,
SPEC.md:563). Expert parameters are TP-sharded with the same G_tensor as the
rest of the model; DTD changes only
*where* rows travel, never the arithmetic, so the oracle has no DTD branch:
G_tensor enters only through the capacity rounding (reading R2).

Precision: every input is decoded exactly (bf16 bit pattern -> fp32 -> fp64)
and every step is carried out in float64. Library primitives used as steps:
numpy matmul (a contraction), exp/tanh, argmax. No blocking, fusion or
reordering beyond the definitions below.

Parity pins: tests/test_oracle_pins.py (brute-force loops, torch-float64
autograd on an independent forward, finite differences, closed forms and
special cases). Every function below is pinned; none is "parity unpinned"
except the absolute output values, for which the paper prints no worked
example.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "decode_bf16", "capacity", "gelu_tanh", "gelu_tanh_grad", "gate", "assign_slots",
    "priority_order", "aux_loss", "aux_loss_dlogits",
    "Routing", "route", "forward_group", "backward_group", "layer",
    "token_forward", "token_backward", "tokens_forward_backward", "expert_row_grads", "TIE_GAP",
]

# BASELINE.json north_star: routing must match bit-exactly "except for logged
# ties whose top-2 logit gap is below 1e-6".
TIE_GAP = 1e-6


def decode_bf16(bits) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64, exactly (16-bit left shift)."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def capacity(tokens: int, experts: int, cf: float, g_tensor: int = 1) -> int:
    """C = ceil(cf * T / E), rounded up to a multiple of G_tensor, at least 1.

    Reading R2: capacity per (token group, expert). The rounding
    to a multiple of G_tensor lets DTD split every expert's C slots into
    G_tensor equal slot slices ("reduces the all-to-all
    message sizes by the degree of tensor parallelism"). Evaluated in double.
    """
    c = int(math.ceil(cf * tokens / experts))
    c = max(c, 1)
    return ((c + g_tensor - 1) // g_tensor) * g_tensor


def gelu_tanh(h: np.ndarray) -> np.ndarray:
    """GeLU, tanh form: 0.5 h (1 + tanh(sqrt(2/pi) (h + 0.044715 h^3))) (reading R8)."""
    u = math.sqrt(2.0 / math.pi) * (h + 0.044715 * h ** 3)
    return 0.5 * h * (1.0 + np.tanh(u))


def gelu_tanh_grad(h: np.ndarray) -> np.ndarray:
    """d gelu_tanh / dh = 0.5 (1 + tanh u) + 0.5 h (1 - tanh^2 u) sqrt(2/pi) (1 + 3*0.044715 h^2)."""
    k = math.sqrt(2.0 / math.pi)
    u = k * (h + 0.044715 * h ** 3)
    th = np.tanh(u)
    return 0.5 * (1.0 + th) + 0.5 * h * (1.0 - th * th) * k * (1.0 + 3.0 * 0.044715 * h * h)


def gate(x: np.ndarray, wg: np.ndarray):
    """Top-1 softmax gate (reading R1, R4).

    l_te = sum_h x_th Wg_he;  e* = lowest index attaining max_e l_te;
    gap = l_max - l_second;   s_te = softmax_e(l_t);  p_t = s_{t, e*}.
    Returns (logits [T,E], expert [T] int32, gap [T], s [T,E], p [T]).
    """
    logits = x @ wg                                   # [T, E] float64
    expert = np.argmax(logits, axis=1).astype(np.int32)   # numpy: first (lowest) max
    T, E = logits.shape
    lmax = logits[np.arange(T), expert]
    if E > 1:
        second = np.partition(logits, E - 2, axis=1)[:, E - 2]
        gap = lmax - second
    else:
        gap = np.full(T, np.inf)
    z = np.exp(logits - lmax[:, None])
    s = z / z.sum(axis=1, keepdims=True)
    p = s[np.arange(T), expert]
    return logits, expert, gap, s, p


def assign_slots(expert: np.ndarray, experts: int, cap: int, order=None):
    """Capacity slots in priority order (reading R3; NEXT #4 random token selection).

    order: the tokens in priority order (a permutation of range(T)); None is
    token order, slot_t = #{t' < t : e*(t') = e*(t)}. In general
    slot_t = #{t' before t in `order` : e*(t') = e*(t)}; kept iff slot_t < C
    (else slot = -1). Returns (slot [T] int32, count [E] kept per expert,
    load [E] routed per expert).
    """
    T = expert.shape[0]
    slot = np.full(T, -1, dtype=np.int32)
    seen = np.zeros(experts, dtype=np.int64)
    for t in (range(T) if order is None else order):
        t = int(t)
        e = int(expert[t])
        if seen[e] < cap:
            slot[t] = seen[e]
        seen[e] += 1
    count = np.minimum(seen, cap).astype(np.int32)
    return slot, count, seen.astype(np.int64)


# --- NEXT #4 gating variants -------------------------------------------------------

_M32 = 0xFFFFFFFF


def _mix32(x: int) -> int:
    """lowbias32 integer hash (the counter-based generator both sides implement)."""
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & _M32
    x ^= x >> 16
    return x


def priority_order(T: int, seed: int) -> np.ndarray:
    """Random token-selection priority (reading R20): order[i] = sigma(i), a keyed
    pseudo-random permutation of range(T) — a 4-round Feistel network on the
    smallest even-width domain 2^(2m) >= T, cycle-walked into [0, T) (a bijection
    of [0, 2^(2m)) restricted by cycle walking stays a bijection of [0, T)).
    Round r: (L, R) -> (R, L ^ (mix32(R ^ k_r) & mask)), k_r = (seed_lo*0x9E3779B9 +
    seed_hi + r*0x85EBCA6B) mod 2^32."""
    if T <= 0:
        return np.zeros(0, dtype=np.int64)
    m = 1
    while (1 << (2 * m)) < T:
        m += 1
    mask = (1 << m) - 1
    lo, hi = seed & _M32, (seed >> 32) & _M32
    keys = [((lo * 0x9E3779B9) + hi + r * 0x85EBCA6B) & _M32 for r in range(4)]

    def feistel(x: int) -> int:
        L, R = x >> m, x & mask
        for k in keys:
            L, R = R, L ^ (_mix32(R ^ k) & mask)
        return (L << m) | R

    out = np.empty(T, dtype=np.int64)
    for i in range(T):
        x = feistel(i)
        while x >= T:
            x = feistel(x)
        out[i] = x
    return out


def aux_loss(expert: np.ndarray, s: np.ndarray, coef: float) -> float:
    """Auxiliary load-balancing loss (reading R21; Switch Transformer eq. 4, GShard):
    l_aux = coef * E * sum_e f_e P_e, f_e = (1/T) #{t : e*(t) = e} (routed, before
    capacity), P_e = (1/T) sum_t s_te."""
    T, E = s.shape
    if T == 0:
        return 0.0
    f = np.bincount(expert, minlength=E) / T
    P = s.mean(axis=0)
    return float(coef * E * np.sum(f * P))


def aux_loss_dlogits(expert: np.ndarray, s: np.ndarray, coef: float) -> np.ndarray:
    """d l_aux / d l_tj with f held constant (it is a count):
    coef * E / T * s_tj (f_j - sum_e f_e s_te), for every token (kept or dropped)."""
    T, E = s.shape
    if T == 0:
        return np.zeros((0, E))
    f = np.bincount(expert, minlength=E) / T
    return coef * E / T * s * (f[None, :] - (s @ f)[:, None])


@dataclass
class Routing:
    logits: np.ndarray
    expert: np.ndarray
    gap: np.ndarray
    s: np.ndarray
    p: np.ndarray
    slot: np.ndarray
    count: np.ndarray
    load: np.ndarray
    cap: int

    @property
    def kept(self) -> np.ndarray:
        return self.slot >= 0


def route(x: np.ndarray, wg: np.ndarray, cap: int, forced=None, override=None, order=None) -> Routing:
    """Gate + slot assignment for one token group.

    forced:   int array [T] — expert ids replacing the argmax for every token
              (the MOE_F_FORCED_ROUTING mode; p is still s_{t, forced}).
    override: (idx, experts) — the tie-override protocol (reading R5): for
              tokens whose top-2 gap is below TIE_GAP the oracle adopts the
              GPU's choice before slots are recomputed.
    order:    priority order of the tokens (priority_order), None = token order.
    """
    logits, expert, gap, s, p = gate(x, wg)
    if forced is not None:
        expert = np.asarray(forced, dtype=np.int32).copy()
    if override is not None:
        idx, ex = override
        expert = expert.copy()
        expert[np.asarray(idx, dtype=np.int64)] = np.asarray(ex, dtype=np.int32)
    p = s[np.arange(s.shape[0]), expert]
    slot, count, load = assign_slots(expert, wg.shape[1], cap, order)
    return Routing(logits, expert, gap, s, p, slot, count, load, cap)


def forward_group(x, wg, w1, w2, r: Routing):
    """Expert FFN + weighted combine for one token group (reading R6, R8).

    For kept token t with expert e: h = x_t W1_e^T, a = gelu_tanh(h),
    o = a W2_e^T, y_t = p_t o. Dropped tokens: y_t = 0.
    x [T,H], wg [H,E], w1 [E,F,H], w2 [E,H,F] all float64.
    Returns (y [T,H], cache) where cache holds per-expert (idx, h, a, o).
    """
    T, H = x.shape
    E = wg.shape[1]
    y = np.zeros((T, H))
    cache = {}
    for e in range(E):
        idx = np.nonzero((r.expert == e) & r.kept)[0]
        if idx.size == 0:
            continue
        h = x[idx] @ w1[e].T
        a = gelu_tanh(h)
        o = a @ w2[e].T
        y[idx] = r.p[idx, None] * o
        cache[e] = (idx, h, a, o)
    return y, cache


def backward_group(x, dy, wg, w1, w2, r: Routing, cache, aux_coef: float = 0.0):
    """Backward of forward_group (reading R6, R13; aux_coef > 0: reading R21).

    do = p dy; dp = <dy, o>; da = do W2_e; dh = da * gelu'(h);
    dx_t = dh W1_e + sum_j dl_tj Wg[:, j], dl_tj = dp_t p_t (delta_{j,e*} - s_tj);
    dW2_e += do^T a; dW1_e += dh^T x_t; dWg += x_t^T dl_t. Dropped tokens: 0.
    Returns (dx [T,H], dwg [H,E], dw1 [E,F,H], dw2 [E,H,F]).
    """
    T, H = x.shape
    E = wg.shape[1]
    dx = np.zeros((T, H))
    dw1 = np.zeros_like(w1)
    dw2 = np.zeros_like(w2)
    dl = np.zeros((T, E))
    for e, (idx, h, a, o) in cache.items():
        do = r.p[idx, None] * dy[idx]
        dp = np.sum(dy[idx] * o, axis=1)
        da = do @ w2[e]
        dh = da * gelu_tanh_grad(h)
        dx[idx] = dh @ w1[e]
        dw2[e] = do.T @ a
        dw1[e] = dh.T @ x[idx]
        onehot = np.zeros((idx.size, E))
        onehot[np.arange(idx.size), e] = 1.0
        dl[idx] = (dp * r.p[idx])[:, None] * (onehot - r.s[idx])
    if aux_coef:
        dl = dl + aux_loss_dlogits(r.expert, r.s, aux_coef)
    dx += dl @ wg.T
    dwg = x.T @ dl
    return dx, dwg, dw1, dw2


def layer(xs, dys, wg, w1, w2, cf: float, g_tensor: int = 1, forced=None, overrides=None,
          priority_seed=None, aux_coef: float = 0.0):
    """The whole layer over S token groups, as one process (no communication).

    xs, dys: lists of S arrays [T,H] (float64). Each group routes its own T
    tokens with its own capacity C (reading R2). Expert weights are global;
    dW1/dW2 sum over every group's tokens (one EP group, G^e_data = 1).
    forced / overrides: per-group lists (or None).
    priority_seed: random token-selection priority (R20), same seed for every group.
    aux_coef: auxiliary load-balancing loss coefficient (R21), per group.
    Returns dict with per-group lists 'y', 'dx', 'dwg', 'routing', 'aux' and summed 'dw1', 'dw2'.
    """
    E = wg.shape[1]
    T = xs[0].shape[0]
    cap = capacity(T, E, cf, g_tensor)
    out = {"y": [], "dx": [], "dwg": [], "routing": [], "aux": [], "cap": cap,
           "dw1": np.zeros_like(w1), "dw2": np.zeros_like(w2)}
    order = None if priority_seed is None else priority_order(T, priority_seed)
    for s, x in enumerate(xs):
        r = route(x, wg, cap,
                  forced=None if forced is None else forced[s],
                  override=None if overrides is None else overrides[s], order=order)
        y, cache = forward_group(x, wg, w1, w2, r)
        out["y"].append(y)
        out["routing"].append(r)
        out["aux"].append(aux_loss(r.expert, r.s, aux_coef))
        if dys is not None:
            dx, dwg, dw1, dw2 = backward_group(x, dys[s], wg, w1, w2, r, cache, aux_coef)
            out["dx"].append(dx)
            out["dwg"].append(dwg)
            out["dw1"] += dw1
            out["dw2"] += dw2
    return out


# --- per-token / per-row evaluation for full-size sampled parity -----------------

def token_forward(t: int, x, w1, w2, r: Routing):
    """y_t and o_t for one token (same definition as forward_group)."""
    if not r.kept[t]:
        return np.zeros(x.shape[1]), None
    e = int(r.expert[t])
    h = w1[e] @ x[t]
    o = w2[e] @ gelu_tanh(h)
    return r.p[t] * o, o


def token_backward(t: int, x, dy, wg, w1, w2, r: Routing):
    """dx_t for one token (same definition as backward_group)."""
    if not r.kept[t]:
        return np.zeros(x.shape[1])
    e = int(r.expert[t])
    h = w1[e] @ x[t]
    o = w2[e] @ gelu_tanh(h)
    dp = float(dy[t] @ o)
    do = r.p[t] * dy[t]
    dh = (do @ w2[e]) * gelu_tanh_grad(h)
    onehot = np.zeros(wg.shape[1])
    onehot[e] = 1.0
    dl = dp * r.p[t] * (onehot - r.s[t])
    return dh @ w1[e] + wg @ dl


def expert_row_grads(e: int, f: int, xs, dys, w1, w2, routings):
    """Row f of dW1_e ([H]) and column f of dW2_e ([H]) summed over all groups.

    dW1_e[f, :] = sum_t dh_tf x_t,  dW2_e[:, f] = sum_t do_t a_tf  over kept
    tokens t of expert e (same definition as backward_group, one f at a time).
    """
    H = xs[0].shape[1]
    g1 = np.zeros(H)
    g2 = np.zeros(H)
    for x, dy, r in zip(xs, dys, routings):
        idx = np.nonzero((r.expert == e) & r.kept)[0]
        if idx.size == 0:
            continue
        hf = x[idx] @ w1[e][f]
        af = gelu_tanh(hf)
        do = r.p[idx, None] * dy[idx]
        dhf = (do @ w2[e][:, f]) * gelu_tanh_grad(hf)
        g1 += dhf @ x[idx]
        g2 += do.T @ af
    return g1, g2


def tokens_forward_backward(idx, x, dy, wg, w1, w2, r: Routing):
    """y_t and dx_t for the tokens `idx` of one group (same definitions as
    forward_group / backward_group, evaluated only for these tokens, one expert at a
    time: h = x_t W1_e^T, a = gelu(h), o = a W2_e^T, y_t = p_t o; dx_t = dh W1_e +
    sum_j dl_tj Wg[:, j] with dl_tj = dp_t p_t (delta_{j,e*} - s_tj); 0 if dropped).
    Returns (y [n, H], dx [n, H])."""
    idx = np.asarray(idx, dtype=np.int64)
    H, E = x.shape[1], wg.shape[1]
    y = np.zeros((idx.size, H))
    dx = np.zeros((idx.size, H))
    for e in range(E):
        sel = np.nonzero((r.expert[idx] == e) & r.kept[idx])[0]
        if sel.size == 0:
            continue
        t = idx[sel]
        h = x[t] @ w1[e].T
        o = gelu_tanh(h) @ w2[e].T
        y[sel] = r.p[t, None] * o
        if dy is None:
            continue
        dp = np.sum(dy[t] * o, axis=1)
        dh = ((r.p[t, None] * dy[t]) @ w2[e]) * gelu_tanh_grad(h)
        onehot = np.zeros((t.size, E))
        onehot[:, e] = 1.0
        dl = (dp * r.p[t])[:, None] * (onehot - r.s[t])
        dx[sel] = dh @ w1[e] + dl @ wg.T
    return y, dx
