"""Pins of the oracle's multi-group branch (S > 1 token groups), CPU only.

With S = G/G_t token groups every expert receives the tokens of every group in
its EP group through the all-to-all: each group
routes its own T tokens with its own softmax gate, its own capacity C and its
own slot order, and the expert-weight gradients are the SUM over groups, while
dx and dWg stay per group. `oracle.moe_oracle.layer` and
`oracle.top2_oracle.layer_top2` implement this by looping over groups; these
tests check that loop against an independent float64 torch forward that
computes the routing itself (argmax, slots by counting) and is differentiated by
autograd, with a separate Wg leaf per group so dWg_s is that group's gradient.

A plausible slip — `dw1 = ...` for `dw1 += ...`, routing group s with group 0's
x, one capacity for all groups, or the priority order of another group — fails
at least one assertion. Capacities under G_tensor rounding are hard-coded values
(reading R2: C = ceil(cf*K*T/E), rounded up to a multiple of G_tensor).
"""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from oracle import top2_oracle as T2


def _groups(S, T, H, F, E, seed, skew=1.0):
    rng = np.random.default_rng(seed)
    xs = [rng.normal(size=(T, H)) for _ in range(S)]
    dys = [rng.normal(size=(T, H)) for _ in range(S)]
    wg = rng.normal(size=(H, E)) / np.sqrt(H)
    wg[:, 0] *= skew
    w1 = rng.normal(size=(E, F, H)) / np.sqrt(H)
    w2 = rng.normal(size=(E, H, F)) / np.sqrt(F)
    return xs, dys, wg, w1, w2


def _slots_by_counting(choices, E, cap, order):
    """choices: list over priority passes of [T] expert ids; slots granted pass by pass, each
    pass in `order` (token ids in priority order). Plain counting loops."""
    T = len(choices[0])
    used = [0] * E
    slot = [[-1] * len(choices) for _ in range(T)]
    for k, ch in enumerate(choices):
        for t in order:
            e = int(ch[t])
            if used[e] < cap:
                slot[t][k] = used[e]
            used[e] += 1
    return slot, [min(u, cap) for u in used]


def _torch_top1(xs, dys, wg, w1, w2, cap, order):
    """Independent top-1 layer over S groups (torch float64, autograd)."""
    W1 = torch.tensor(w1, requires_grad=True)
    W2 = torch.tensor(w2, requires_grad=True)
    out = {"y": [], "dx": [], "dwg": [], "slot": [], "count": []}
    leaves = []
    total = 0.0
    for x, dy in zip(xs, dys):
        X = torch.tensor(x, requires_grad=True)
        WG = torch.tensor(wg, requires_grad=True)
        logits = X @ WG
        expert = torch.argmax(logits.detach(), dim=1).numpy()   # first maximum = lowest index
        slot, count = _slots_by_counting([expert], wg.shape[1], cap, order)
        s = torch.softmax(logits, dim=1)
        rows = []
        for t in range(x.shape[0]):
            e = int(expert[t])
            if slot[t][0] < 0:
                rows.append(torch.zeros(x.shape[1], dtype=torch.float64))
                continue
            a = torch.nn.functional.gelu(W1[e] @ X[t], approximate="tanh")
            rows.append(s[t, e] * (W2[e] @ a))
        y = torch.stack(rows)
        total = total + (y * torch.tensor(dy)).sum()
        out["y"].append(y.detach().numpy())
        out["slot"].append(np.array([sl[0] for sl in slot]))
        out["count"].append(np.array(count))
        leaves.append((X, WG))
    total.backward()
    out["dx"] = [X.grad.numpy() for X, _ in leaves]
    out["dwg"] = [WG.grad.numpy() for _, WG in leaves]
    out["dw1"], out["dw2"] = W1.grad.numpy(), W2.grad.numpy()
    return out


@pytest.mark.parametrize("S,T,E,cf,gt,cap,skew,seed", [
    (2, 24, 4, 1.0, 1, 6, 1.0, 0),    # ceil(24/4) = 6
    (3, 21, 4, 1.0, 1, 6, 1.0, 1),    # ceil(5.25) = 6
    (3, 37, 4, 0.5, 2, 6, 2.0, 2),    # ceil(4.625) = 5 -> 6 (multiple of G_t = 2); drop-heavy
    (2, 37, 4, 0.5, 4, 8, 2.0, 3),    # 5 -> 8 (multiple of 4)
    (2, 30, 5, 0.25, 4, 4, 3.0, 4),   # ceil(1.5) = 2 -> 4; expert 0 oversubscribed
])
def test_layer_multigroup_matches_torch_autograd(S, T, E, cf, gt, cap, skew, seed):
    H, F = 8, 12
    xs, dys, wg, w1, w2 = _groups(S, T, H, F, E, seed, skew)
    out = O.layer(xs, dys, wg, w1, w2, cf, g_tensor=gt)
    assert out["cap"] == cap
    ref = _torch_top1(xs, dys, wg, w1, w2, cap, list(range(T)))
    for s in range(S):
        r = out["routing"][s]
        np.testing.assert_array_equal(r.slot, ref["slot"][s])
        np.testing.assert_array_equal(r.count, ref["count"][s])
        np.testing.assert_allclose(out["y"][s], ref["y"][s], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(out["dx"][s], ref["dx"][s], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(out["dwg"][s], ref["dwg"][s], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw1"], ref["dw1"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw2"], ref["dw2"], rtol=1e-9, atol=1e-12)
    if cf < 1:
        assert any((~r.kept).any() for r in out["routing"]), "drop-heavy case must drop tokens"
    # the groups really differ (a group-0-for-all slip would be invisible otherwise)
    assert any(not np.array_equal(out["routing"][0].slot, out["routing"][s].slot) for s in range(1, S))


def test_layer_multigroup_sum_is_not_last_group():
    """dW1/dW2 over S groups equal the sum of the single-group oracles, and differ from
    any one group's gradient (guards `=` for `+=`)."""
    xs, dys, wg, w1, w2 = _groups(3, 20, 8, 12, 4, seed=11)
    out = O.layer(xs, dys, wg, w1, w2, 1.0)
    singles = [O.layer([x], [dy], wg, w1, w2, 1.0) for x, dy in zip(xs, dys)]
    np.testing.assert_allclose(out["dw1"], sum(o["dw1"] for o in singles), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(out["dw2"], sum(o["dw2"] for o in singles), rtol=1e-12, atol=1e-14)
    for o in singles:
        assert np.abs(out["dw1"] - o["dw1"]).max() > 1e-3


def test_layer_multigroup_priority_order():
    """Random token selection (R20): every group uses the same keyed order over its own
    tokens; slots follow that order, per group."""
    S, T, E = 2, 33, 4
    xs, dys, wg, w1, w2 = _groups(S, T, 8, 12, E, seed=21, skew=2.0)
    seed = 987654321
    out = O.layer(xs, dys, wg, w1, w2, 0.5, g_tensor=2, priority_seed=seed)
    order = [int(t) for t in O.priority_order(T, seed)]
    assert sorted(order) == list(range(T)) and order != list(range(T))
    ref = _torch_top1(xs, dys, wg, w1, w2, out["cap"], order)
    assert out["cap"] == 6   # ceil(0.5*33/4) = 5 -> 6
    for s in range(S):
        np.testing.assert_array_equal(out["routing"][s].slot, ref["slot"][s])
        np.testing.assert_allclose(out["dx"][s], ref["dx"][s], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(out["dwg"][s], ref["dwg"][s], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw1"], ref["dw1"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw2"], ref["dw2"], rtol=1e-9, atol=1e-12)


def _torch_top2(xs, dys, wg, w1, w2, cap, order):
    """Independent top-2 layer over S groups (GShard renormalised pair, R22)."""
    W1 = torch.tensor(w1, requires_grad=True)
    W2 = torch.tensor(w2, requires_grad=True)
    out = {"y": [], "slot": []}
    leaves = []
    total = 0.0
    E = wg.shape[1]
    for x, dy in zip(xs, dys):
        X = torch.tensor(x, requires_grad=True)
        WG = torch.tensor(wg, requires_grad=True)
        logits = X @ WG
        ld = logits.detach().numpy()
        e1 = [max(range(E), key=lambda j: (ld[t, j], -j)) for t in range(x.shape[0])]
        e2 = [max((j for j in range(E) if j != e1[t]), key=lambda j: (ld[t, j], -j))
              for t in range(x.shape[0])]
        slot, _ = _slots_by_counting([e1, e2], E, cap, order)
        s = torch.softmax(logits, dim=1)
        rows = []
        for t in range(x.shape[0]):
            pair = (e1[t], e2[t])
            S_ = s[t, pair[0]] + s[t, pair[1]]
            yt = torch.zeros(x.shape[1], dtype=torch.float64)
            for k in range(2):
                if slot[t][k] < 0:
                    continue
                a = torch.nn.functional.gelu(W1[pair[k]] @ X[t], approximate="tanh")
                yt = yt + (s[t, pair[k]] / S_) * (W2[pair[k]] @ a)
            rows.append(yt)
        y = torch.stack(rows)
        total = total + (y * torch.tensor(dy)).sum()
        out["y"].append(y.detach().numpy())
        out["slot"].append(np.array(slot))
        leaves.append((X, WG))
    total.backward()
    out["dx"] = [X.grad.numpy() for X, _ in leaves]
    out["dwg"] = [WG.grad.numpy() for _, WG in leaves]
    out["dw1"], out["dw2"] = W1.grad.numpy(), W2.grad.numpy()
    return out


@pytest.mark.parametrize("S,T,E,cf,gt,cap,seed,prio", [
    (2, 20, 4, 1.0, 1, 10, 0, None),   # ceil(2*20/4) = 10
    (3, 19, 5, 0.5, 2, 4, 1, None),    # ceil(0.5*38/5) = 4 (already even)
    (2, 23, 4, 0.5, 4, 8, 2, 77),      # ceil(5.75) = 6 -> 8; random priority
])
def test_layer_top2_multigroup_matches_torch_autograd(S, T, E, cf, gt, cap, seed, prio):
    xs, dys, wg, w1, w2 = _groups(S, T, 8, 12, E, seed, skew=2.0)
    order = None if prio is None else O.priority_order(T, prio)
    out = T2.layer_top2(xs, dys, wg, w1, w2, cf, gt, order=order)
    assert out["cap"] == cap
    ref = _torch_top2(xs, dys, wg, w1, w2, cap, list(range(T)) if order is None else [int(t) for t in order])
    for s in range(S):
        np.testing.assert_array_equal(out["routing"][s].slot, ref["slot"][s])
        np.testing.assert_allclose(out["y"][s], ref["y"][s], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(out["dx"][s], ref["dx"][s], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(out["dwg"][s], ref["dwg"][s], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw1"], ref["dw1"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw2"], ref["dw2"], rtol=1e-9, atol=1e-12)
    singles = [T2.layer_top2([x], [dy], wg, w1, w2, cf, gt, order=order)["dw1"] for x, dy in zip(xs, dys)]
    for d1 in singles:
        assert np.abs(out["dw1"] - d1).max() > 1e-3
