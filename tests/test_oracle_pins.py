"""Pins for the CPU oracle against things other than itself (CPU only).

Each pin is chosen so a plausible slip in oracle/moe_oracle.py (a dropped
term, a wrong sign or index, a transposed operand) fails at least one test:
  * brute-force pure-Python loops of the definitions on tiny inputs,
  * an independent float64 torch forward differentiated by autograd
    (pins every backward formula),
  * central finite differences,
  * library routines for special cases (E = 1 -> dense GeLU MLP via
    torch.nn.functional.linear/gelu),
  * closed forms (x = 0 routing, gelu odd-part identity, capacity values).
"""
import math

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2305_13525_b200 import synth


def _tiny(T=24, H=8, F=6, E=3, seed=0):
    g = np.random.default_rng(seed)
    x = g.standard_normal((T, H))
    wg = g.standard_normal((H, E)) / math.sqrt(H)
    w1 = g.standard_normal((E, F, H)) / math.sqrt(H)
    w2 = g.standard_normal((E, H, F)) / math.sqrt(F)
    dy = g.standard_normal((T, H))
    return x, wg, w1, w2, dy


# ---------------------------------------------------------------- capacity
@pytest.mark.parametrize("T,E,cf,gt,want", [
    (256, 4, 1.0, 1, 64),          # BASELINE tiny config
    (16384, 16, 1.0, 1, 1024),     # 1.3B config
    (16384, 32, 1.0, 1, 512),      # 2.7B config
    (16384, 16, 1.0, 2, 1024),     # 6.7B config (already a multiple of 2)
    (100, 3, 1.0, 4, 36),          # ceil(33.33)=34 -> next multiple of 4
    (10, 4, 1.25, 1, 4),           # ceil(3.125)
    (1, 8, 1.0, 1, 1),             # minimum 1
    (0, 8, 1.0, 2, 2),             # empty input still gets >= 1 slot, rounded to G_t
])
def test_capacity_closed_form(T, E, cf, gt, want):
    assert O.capacity(T, E, cf, gt) == want


# ---------------------------------------------------------------- gelu
def test_gelu_matches_torch_tanh_gelu():
    h = np.linspace(-8, 8, 2001)
    ref = torch.nn.functional.gelu(torch.tensor(h, dtype=torch.float64), approximate="tanh").numpy()
    np.testing.assert_allclose(O.gelu_tanh(h), ref, rtol=1e-13, atol=1e-15)


def test_gelu_odd_part_identity_and_zero():
    h = np.linspace(-5, 5, 101)
    np.testing.assert_allclose(O.gelu_tanh(h) - O.gelu_tanh(-h), h, atol=1e-13)
    assert O.gelu_tanh(np.array([0.0]))[0] == 0.0
    assert O.gelu_tanh_grad(np.array([0.0]))[0] == 0.5


def test_gelu_grad_finite_difference_and_autograd():
    h = np.linspace(-6, 6, 241)
    eps = 1e-6
    fd = (O.gelu_tanh(h + eps) - O.gelu_tanh(h - eps)) / (2 * eps)
    np.testing.assert_allclose(O.gelu_tanh_grad(h), fd, atol=1e-8)
    ht = torch.tensor(h, dtype=torch.float64, requires_grad=True)
    torch.nn.functional.gelu(ht, approximate="tanh").sum().backward()
    np.testing.assert_allclose(O.gelu_tanh_grad(h), ht.grad.numpy(), atol=1e-13)


# ---------------------------------------------------------------- gate
def _gate_bruteforce(x, wg):
    T, H = x.shape
    E = wg.shape[1]
    res = []
    for t in range(T):
        l = [sum(float(x[t, h]) * float(wg[h, e]) for h in range(H)) for e in range(E)]
        best = 0
        for e in range(1, E):
            if l[e] > l[best]:
                best = e
        rest = sorted(l, reverse=True)
        gap = rest[0] - rest[1] if E > 1 else math.inf
        m = max(l)
        z = [math.exp(v - m) for v in l]
        p = z[best] / sum(z)
        res.append((l, best, gap, p))
    return res


def test_gate_bruteforce_tiny():
    x, wg, *_ = _tiny(T=20, H=7, E=5)
    logits, expert, gap, s, p = O.gate(x, wg)
    for t, (l, best, g, pp) in enumerate(_gate_bruteforce(x, wg)):
        np.testing.assert_allclose(logits[t], l, rtol=1e-12, atol=1e-14)
        assert expert[t] == best
        assert abs(gap[t] - g) < 1e-12
        assert abs(p[t] - pp) < 1e-14
    np.testing.assert_allclose(s.sum(axis=1), 1.0, atol=1e-14)


def test_gate_zero_tokens_route_to_expert0_uniform():
    x = np.zeros((9, 4))
    wg = np.random.default_rng(1).standard_normal((4, 6))
    logits, expert, gap, s, p = O.gate(x, wg)
    assert (expert == 0).all()
    np.testing.assert_allclose(p, 1.0 / 6, atol=0)
    assert (gap == 0).all()


def test_gate_single_expert_prob_one():
    x, wg, *_ = _tiny(E=1)
    _, expert, gap, _, p = O.gate(x, wg[:, :1])
    assert (expert == 0).all() and (p == 1.0).all() and np.isinf(gap).all()


def test_gate_exact_tie_lowest_index():
    x, wg, *_ = _tiny(E=4)
    wg = wg.copy()
    wg[:, 3] = wg[:, 1]                 # columns 1 and 3 identical -> exact ties
    logits, expert, gap, _, _ = O.gate(x, wg)
    tie = logits[:, 1] == logits.max(axis=1)
    assert tie.any()
    assert (expert[tie] == 1).all() and (gap[tie] == 0).all()


# ---------------------------------------------------------------- slots
def test_slots_bruteforce_definition():
    g = np.random.default_rng(3)
    for trial in range(20):
        T, E = int(g.integers(1, 60)), int(g.integers(1, 7))
        expert = g.integers(0, E, T).astype(np.int32)
        C = int(g.integers(1, 12))
        slot, count, load = O.assign_slots(expert, E, C)
        for t in range(T):
            before = sum(1 for u in range(t) if expert[u] == expert[t])
            assert slot[t] == (before if before < C else -1)
        for e in range(E):
            n = int((expert == e).sum())
            assert load[e] == n and count[e] == min(n, C) <= C
            kept = np.nonzero((expert == e) & (slot >= 0))[0]
            assert list(kept) == list(np.nonzero(expert == e)[0][:C])
        assert load.sum() == T


def test_route_override_recomputes_slots():
    x, wg, *_ = _tiny(T=30, E=3)
    r0 = O.route(x, wg, cap=5)
    t = int(np.nonzero(r0.kept)[0][0])
    new_e = (int(r0.expert[t]) + 1) % 3
    r1 = O.route(x, wg, cap=5, override=([t], [new_e]))
    assert r1.expert[t] == new_e
    ref_slot, _, _ = O.assign_slots(r1.expert, 3, 5)
    np.testing.assert_array_equal(r1.slot, ref_slot)
    assert abs(r1.p[t] - r1.s[t, new_e]) == 0


# ---------------------------------------------------------------- forward
def _forward_bruteforce(x, wg, w1, w2, cap):
    T, H = x.shape
    E, F, _ = w1.shape
    gates = _gate_bruteforce(x, wg)
    seen = [0] * E
    y = [[0.0] * H for _ in range(T)]
    for t in range(T):
        _, e, _, p = gates[t]
        if seen[e] < cap:
            hvec = [sum(w1[e, f, k] * x[t, k] for k in range(H)) for f in range(F)]
            avec = [0.5 * v * (1 + math.tanh(math.sqrt(2 / math.pi) * (v + 0.044715 * v ** 3))) for v in hvec]
            for k in range(H):
                y[t][k] = p * sum(w2[e, k, f] * avec[f] for f in range(F))
        seen[e] += 1
    return np.array(y)


@pytest.mark.parametrize("cap", [2, 4, 100])
def test_forward_bruteforce_tiny(cap):
    x, wg, w1, w2, _ = _tiny(T=18, H=6, F=5, E=3)
    r = O.route(x, wg, cap)
    y, _ = O.forward_group(x, wg, w1, w2, r)
    np.testing.assert_allclose(y, _forward_bruteforce(x, wg, w1, w2, cap), rtol=1e-12, atol=1e-13)
    assert (y[~r.kept] == 0).all()


def test_single_expert_is_dense_gelu_mlp():
    x, wg, w1, w2, _ = _tiny(T=40, H=16, F=24, E=1)
    cap = O.capacity(40, 1, 1.0)
    r = O.route(x, wg, cap)
    y, _ = O.forward_group(x, wg, w1, w2, r)
    xt = torch.tensor(x)
    ref = torch.nn.functional.linear(
        torch.nn.functional.gelu(torch.nn.functional.linear(xt, torch.tensor(w1[0])), approximate="tanh"),
        torch.tensor(w2[0]))
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- backward
def _torch_layer_loss(x, wg, w1, w2, dy, expert, kept):
    """Independent float64 torch forward with the discrete routing held fixed;
    autograd then differentiates it (pins every hand-derived backward term)."""
    s = torch.softmax(x @ wg, dim=1)
    p = s[torch.arange(x.shape[0]), expert]
    y = torch.zeros_like(x)
    for e in range(wg.shape[1]):
        m = (expert == e) & kept
        if m.any():
            h = x[m] @ w1[e].T
            o = torch.nn.functional.gelu(h, approximate="tanh") @ w2[e].T
            y = y.index_put((m.nonzero()[:, 0],), p[m, None] * o)
    return (y * dy).sum()


@pytest.mark.parametrize("cap", [3, 50])
def test_backward_matches_torch_autograd(cap):
    x, wg, w1, w2, dy = _tiny(T=30, H=10, F=7, E=4, seed=5)
    r = O.route(x, wg, cap)
    y, cache = O.forward_group(x, wg, w1, w2, r)
    dx, dwg, dw1, dw2 = O.backward_group(x, dy, wg, w1, w2, r, cache)
    ts = [torch.tensor(a, requires_grad=True) for a in (x, wg, w1, w2)]
    loss = _torch_layer_loss(*ts, torch.tensor(dy), torch.tensor(r.expert.astype(np.int64)),
                             torch.tensor(r.kept))
    loss.backward()
    for mine, t in zip((dx, dwg, dw1, dw2), ts):
        np.testing.assert_allclose(mine, t.grad.numpy(), rtol=1e-10, atol=1e-12)
    assert (dx[~r.kept] == 0).all()


def test_backward_finite_difference():
    x, wg, w1, w2, dy = _tiny(T=16, H=5, F=4, E=3, seed=9)
    cap = 4
    r = O.route(x, wg, cap)
    assert (r.gap > 1e-3).all()
    y, cache = O.forward_group(x, wg, w1, w2, r)
    dx, dwg, dw1, dw2 = O.backward_group(x, dy, wg, w1, w2, r, cache)

    def loss(x_, wg_, w1_, w2_):
        rr = O.route(x_, wg_, cap, forced=r.expert)     # routing held fixed
        yy, _ = O.forward_group(x_, wg_, w1_, w2_, rr)
        return float((yy * dy).sum())

    eps = 1e-6
    args = [x, wg, w1, w2]
    for which, grad in enumerate((dx, dwg, dw1, dw2)):
        g = np.random.default_rng(which)
        for _ in range(6):
            idx = tuple(int(g.integers(0, n)) for n in args[which].shape)
            plus = [a.copy() for a in args]
            minus = [a.copy() for a in args]
            plus[which][idx] += eps
            minus[which][idx] -= eps
            fd = (loss(*plus) - loss(*minus)) / (2 * eps)
            assert abs(fd - grad[idx]) < 1e-6 * max(1.0, abs(fd)), (which, idx, fd, grad[idx])


def test_dropped_tokens_zero_and_all_to_one():
    x, wg, w1, w2, dy = _tiny(T=20, E=4)
    forced = np.zeros(20, dtype=np.int32)
    out = O.layer([x], [dy], wg, w1, w2, cf=1.0, forced=[forced])
    r = out["routing"][0]
    assert r.count[0] == out["cap"] == 5 and r.kept.sum() == 5
    assert (out["y"][0][5:] == 0).all() and (out["dx"][0][5:] == 0).all()
    assert (out["dw1"][1:] == 0).all() and (out["dw2"][1:] == 0).all()


def test_per_token_and_row_helpers_match_full():
    shape = synth.CONFIGS["tiny"]
    x = O.decode_bf16(synth.make_x(shape))
    dy = O.decode_bf16(synth.make_dy(shape))
    wg = synth.make_wg(shape).astype(np.float64)
    w1b, w2b = synth.make_experts(shape)
    w1, w2 = O.decode_bf16(w1b), O.decode_bf16(w2b)
    out = O.layer([x], [dy], wg, w1, w2, cf=1.0)
    r = out["routing"][0]
    for t in (0, 7, 100, 255):
        yt, _ = O.token_forward(t, x, w1, w2, r)
        np.testing.assert_allclose(yt, out["y"][0][t], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(O.token_backward(t, x, dy, wg, w1, w2, r), out["dx"][0][t],
                                   rtol=1e-10, atol=1e-12)
    for e, f in ((0, 0), (3, 255), (2, 17)):
        g1, g2 = O.expert_row_grads(e, f, [x], [dy], w1, w2, [r])
        np.testing.assert_allclose(g1, out["dw1"][e][f], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g2, out["dw2"][e][:, f], rtol=1e-10, atol=1e-12)


def test_bf16_decode_exact():
    vals = np.array([0.0, 1.0, -2.5, 3.140625, 1e-3], dtype=np.float32)
    bits = synth.f32_to_bf16_bits(vals)
    ref = torch.tensor(vals).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(O.decode_bf16(bits), ref)


def test_tokens_forward_backward_matches_full_layer():
    """The subset evaluation used by the full-size sampled parity equals the full layer on
    every token it is asked for (kept and dropped), in any order, with repeats."""
    x, wg, w1, w2, dy = _tiny(T=40, H=8, F=6, E=4, seed=13)
    r = O.route(x, wg, cap=7)
    y, cache = O.forward_group(x, wg, w1, w2, r)
    dx, *_ = O.backward_group(x, dy, wg, w1, w2, r, cache)
    assert (~r.kept).any()
    idx = np.array([39, 0, 5, 5, 17, *np.nonzero(~r.kept)[0][:3]])
    ys, dxs = O.tokens_forward_backward(idx, x, dy, wg, w1, w2, r)
    np.testing.assert_allclose(ys, y[idx], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dxs, dx[idx], rtol=1e-10, atol=1e-12)
