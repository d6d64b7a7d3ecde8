"""Pins of oracle/top2_oracle.py (reading R22, NEXT #4 top-2 gating), CPU:
brute-force loops, torch float64 autograd of an independent forward, and
special cases where the gate must drop out of the result."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from oracle import top2_oracle as T2


def _problem(T=24, H=8, F=12, E=4, seed=0, skew=1.0):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(T, H))
    dy = rng.normal(size=(T, H))
    wg = rng.normal(size=(H, E)) / np.sqrt(H)
    wg[:, 0] *= skew
    w1 = rng.normal(size=(E, F, H)) / np.sqrt(H)
    w2 = rng.normal(size=(E, H, F)) / np.sqrt(F)
    return x, dy, wg, w1, w2


def test_capacity_top2():
    assert T2.capacity_top2(16384, 16, 1.0) == 2048
    assert T2.capacity_top2(256, 4, 1.0, 2) == 128
    assert T2.capacity_top2(10, 4, 0.5, 4) == 4     # ceil(2.5) = 3 -> multiple of 4
    assert T2.capacity_top2(1, 64, 0.01) == 1


def test_gate_top2_brute_force():
    x, _, wg, _, _ = _problem(T=40, E=6, seed=1)
    logits, experts, gap, s, w = T2.gate_top2(x, wg)
    for t in range(40):
        l = [float(x[t] @ wg[:, j]) for j in range(6)]
        e1 = max(range(6), key=lambda j: (l[j], -j))
        e2 = max((j for j in range(6) if j != e1), key=lambda j: (l[j], -j))
        assert (experts[t] == [e1, e2]).all()
        rest = sorted(l, reverse=True)
        assert gap[t] == pytest.approx(min(rest[0] - rest[1], rest[1] - rest[2]))
        z = np.exp(np.array(l) - max(l))
        p = z / z.sum()
        assert w[t, 0] == pytest.approx(p[e1] / (p[e1] + p[e2]))
        assert w[t].sum() == pytest.approx(1.0)


def test_exact_ties_lowest_indices():
    x = np.ones((3, 2))
    wg = np.zeros((2, 5))
    wg[:, 1] = wg[:, 3] = 1.0  # experts 1 and 3 tie for first; 0, 2, 4 tie for third
    _, experts, gap, _, _ = T2.gate_top2(x, wg)
    assert (experts == [1, 3]).all()
    assert (gap == 0).all()


def test_slots_brute_force():
    rng = np.random.default_rng(4)
    T, E = 50, 4
    for trial in range(5):
        experts = np.stack([rng.integers(0, E, T), rng.integers(0, E, T)], axis=1).astype(np.int32)
        cap = int(rng.integers(1, 30))
        order = O.priority_order(T, trial) if trial % 2 else None
        slot, count, load = T2.assign_slots_top2(experts, E, cap, order)
        seq = list(range(T)) if order is None else list(order)
        pos = {t: i for i, t in enumerate(seq)}
        for t in range(T):
            for k in range(2):
                e = experts[t, k]
                n = sum(1 for u in range(T) if experts[u, 0] == e and (k == 1 or pos[u] < pos[t]))
                if k == 1:
                    n += sum(1 for u in range(T) if experts[u, 1] == e and pos[u] < pos[t])
                assert slot[t, k] == (n if n < cap else -1)
        np.testing.assert_array_equal(load, np.bincount(experts.reshape(-1), minlength=E))
        np.testing.assert_array_equal(count, np.minimum(load, cap))


def _torch_layer(x, dy, wg, w1, w2, r):
    """Independent top-2 forward in torch float64, differentiated by autograd; routing
    (choices and kept flags) taken from r as constants."""
    X = torch.tensor(x, requires_grad=True)
    WG = torch.tensor(wg, requires_grad=True)
    W1 = torch.tensor(w1, requires_grad=True)
    W2 = torch.tensor(w2, requires_grad=True)
    s = torch.softmax(X @ WG, dim=1)
    T = x.shape[0]
    ys = []
    for t in range(T):
        e = [int(r.experts[t, 0]), int(r.experts[t, 1])]
        S = s[t, e[0]] + s[t, e[1]]
        yt = torch.zeros(x.shape[1], dtype=torch.float64)
        for k in range(2):
            if r.slot[t, k] < 0:
                continue
            h = W1[e[k]] @ X[t]
            a = torch.nn.functional.gelu(h, approximate="tanh")
            yt = yt + (s[t, e[k]] / S) * (W2[e[k]] @ a)
        ys.append(yt)
    y = torch.stack(ys)
    (y * torch.tensor(dy)).sum().backward()
    return y.detach().numpy(), X.grad.numpy(), WG.grad.numpy(), W1.grad.numpy(), W2.grad.numpy()


@pytest.mark.parametrize("seed,cf,skew", [(0, 4.0, 1.0), (1, 1.0, 1.0), (2, 0.5, 2.0), (3, 0.25, 3.0)])
def test_layer_matches_torch_autograd(seed, cf, skew):
    x, dy, wg, w1, w2 = _problem(seed=seed, skew=skew)
    out = T2.layer_top2([x], [dy], wg, w1, w2, cf)
    r = out["routing"][0]
    if cf < 1:
        assert (~r.kept).any()
    y, dx, dwg, dw1, dw2 = _torch_layer(x, dy, wg, w1, w2, r)
    np.testing.assert_allclose(out["y"][0], y, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(out["dx"][0], dx, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dwg"][0], dwg, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw1"], dw1, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["dw2"], dw2, rtol=1e-9, atol=1e-12)


def test_identical_experts_gate_drops_out():
    """Every expert the same and nothing dropped: y_t = FFN(x_t) whatever the gate, since the
    two renormalised weights sum to 1 -> dWg = 0 and the gate term of dx vanishes."""
    x, dy, wg, w1, w2 = _problem(T=30, E=5, seed=6)
    w1[:] = w1[0]
    w2[:] = w2[0]
    out = T2.layer_top2([x], [dy], wg, w1, w2, 8.0)
    assert out["routing"][0].kept.all()
    ffn = O.gelu_tanh(x @ w1[0].T) @ w2[0].T
    np.testing.assert_allclose(out["y"][0], ffn, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out["dwg"][0], 0.0, atol=1e-12)


def test_two_experts_both_always_chosen():
    x, dy, wg, w1, w2 = _problem(T=20, E=2, seed=7)
    r = T2.layer_top2([x], [dy], wg, w1, w2, 1.0)["routing"][0]
    assert (np.sort(r.experts, axis=1) == [0, 1]).all()
    np.testing.assert_allclose(r.w.sum(axis=1), 1.0)
