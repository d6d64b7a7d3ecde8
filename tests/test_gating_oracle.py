"""Pins of the NEXT #4 gating variants in oracle/moe_oracle.py (CPU):
random token-selection priority (reading R20) and the auxiliary load-balancing
loss (reading R21) — against brute force, invariants, closed forms and torch
float64 autograd on an independent implementation."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O


# ---------------------------------------------------------------- priority permutation
@pytest.mark.parametrize("T", list(range(1, 70)) + [255, 256, 257, 1000, 4096, 4097, 16384])
def test_priority_order_is_a_permutation(T):
    o = O.priority_order(T, 0xC0FFEE)
    assert o.shape == (T,)
    np.testing.assert_array_equal(np.sort(o), np.arange(T))


def test_priority_order_keyed_and_deterministic():
    a = O.priority_order(1000, 1)
    np.testing.assert_array_equal(a, O.priority_order(1000, 1))
    assert not np.array_equal(a, O.priority_order(1000, 2))
    assert not np.array_equal(a, O.priority_order(1000, 1 << 32))  # the high key word matters
    assert not np.array_equal(a, np.arange(1000))


def test_priority_order_roughly_uniform():
    """Position of token 0 over 2000 keys, T = 8: chi-square against uniform."""
    T, n = 8, 2000
    hits = np.zeros(T)
    for seed in range(n):
        hits[int(np.nonzero(O.priority_order(T, seed) == 0)[0][0])] += 1
    chi2 = ((hits - n / T) ** 2 / (n / T)).sum()
    assert chi2 < 30.0, (hits, chi2)  # 7 d.o.f.: P(chi2 > 24.3) = 0.001


# ---------------------------------------------------------------- slots in priority order
def _slots_brute(expert, E, cap, order):
    pos = np.empty(len(order), dtype=np.int64)
    pos[np.asarray(order)] = np.arange(len(order))
    slot = np.full(len(expert), -1)
    for t in range(len(expert)):
        before = sum(1 for u in range(len(expert)) if expert[u] == expert[t] and pos[u] < pos[t])
        if before < cap:
            slot[t] = before
    return slot


@pytest.mark.parametrize("seed", range(6))
def test_assign_slots_priority_brute_force(seed):
    rng = np.random.default_rng(seed)
    T, E = 60, 4
    expert = rng.integers(0, E, T).astype(np.int32)
    cap = int(rng.integers(1, 20))
    order = O.priority_order(T, seed)
    slot, count, load = O.assign_slots(expert, E, cap, order)
    np.testing.assert_array_equal(slot, _slots_brute(expert, E, cap, order))
    np.testing.assert_array_equal(load, np.bincount(expert, minlength=E))
    np.testing.assert_array_equal(count, np.minimum(load, cap))
    assert (slot < cap).all()


def test_identity_order_is_token_order():
    rng = np.random.default_rng(3)
    expert = rng.integers(0, 5, 200).astype(np.int32)
    a = O.assign_slots(expert, 5, 17)
    b = O.assign_slots(expert, 5, 17, np.arange(200))
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


def test_random_priority_drops_differ_from_token_order():
    """With every token on one expert, token order keeps the first C tokens; random
    priority keeps the first C of the permutation."""
    T, cap = 100, 10
    expert = np.zeros(T, np.int32)
    slot_tok = O.assign_slots(expert, 2, cap)[0]
    order = O.priority_order(T, 9)
    slot_rts = O.assign_slots(expert, 2, cap, order)[0]
    np.testing.assert_array_equal(np.nonzero(slot_tok >= 0)[0], np.arange(cap))
    np.testing.assert_array_equal(np.sort(np.nonzero(slot_rts >= 0)[0]), np.sort(order[:cap]))
    np.testing.assert_array_equal(slot_rts[order[:cap]], np.arange(cap))


# ---------------------------------------------------------------- aux loss
def test_aux_loss_uniform_gate_closed_form():
    """Wg = 0: s_te = 1/E and every token picks expert 0 (lowest index) ->
    f = (1, 0, ...), P = 1/E -> l_aux = coef * E * 1/E = coef."""
    x = np.random.default_rng(0).normal(size=(64, 16))
    r = O.route(x, np.zeros((16, 4)), 64)
    assert O.aux_loss(r.expert, r.s, 0.01) == pytest.approx(0.01, rel=1e-12)


def test_aux_loss_balanced_minimum():
    """f_e = P_e = 1/E (balanced one-hot-ish routing) -> l_aux = coef (the minimum of
    E sum f P over a balanced f)."""
    E, T = 4, 400
    expert = np.repeat(np.arange(E), T // E).astype(np.int32)
    s = np.full((T, E), 1.0 / E)
    assert O.aux_loss(expert, s, 0.5) == pytest.approx(0.5, rel=1e-12)


def test_aux_dlogits_matches_torch_autograd():
    rng = np.random.default_rng(5)
    T, H, E, coef = 50, 12, 6, 0.03
    x = rng.normal(size=(T, H))
    wg = rng.normal(size=(H, E)) / np.sqrt(H)
    logits = torch.tensor(x @ wg, dtype=torch.float64, requires_grad=True)
    s = torch.softmax(logits, dim=1)
    expert = torch.argmax(logits.detach(), dim=1)
    f = torch.bincount(expert, minlength=E).double() / T           # a count: constant
    loss = coef * E * (f * s.mean(dim=0)).sum()
    loss.backward()
    r = O.route(x, wg, T)
    assert O.aux_loss(r.expert, r.s, coef) == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(O.aux_loss_dlogits(r.expert, r.s, coef), logits.grad.numpy(),
                               rtol=1e-10, atol=1e-15)


def test_layer_aux_gradient_terms():
    """The layer backward adds exactly x^T dl_aux to dWg and dl_aux Wg^T to dx — for
    every token, dropped ones included (which otherwise get dx = 0)."""
    rng = np.random.default_rng(8)
    T, H, F, E, coef = 40, 16, 24, 4, 0.05
    x = rng.normal(size=(T, H))
    dy = rng.normal(size=(T, H))
    wg = rng.normal(size=(H, E)) / np.sqrt(H)
    wg[:, 0] *= 3.0  # oversubscribe expert 0: drops
    w1 = rng.normal(size=(E, F, H)) / np.sqrt(H)
    w2 = rng.normal(size=(E, H, F)) / np.sqrt(F)
    base = O.layer([x], [dy], wg, w1, w2, 0.5)
    aux = O.layer([x], [dy], wg, w1, w2, 0.5, aux_coef=coef)
    r = aux["routing"][0]
    assert (~r.kept).any()
    dl = O.aux_loss_dlogits(r.expert, r.s, coef)
    np.testing.assert_allclose(aux["dwg"][0] - base["dwg"][0], x.T @ dl, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(aux["dx"][0] - base["dx"][0], dl @ wg.T, rtol=1e-10, atol=1e-14)
    assert np.abs(aux["dx"][0][~r.kept]).max() > 0
    assert (base["dx"][0][~r.kept] == 0).all()
    np.testing.assert_array_equal(aux["y"][0], base["y"][0])  # the loss is a side output
    assert aux["aux"][0] == pytest.approx(O.aux_loss(r.expert, r.s, coef))


def test_layer_aux_dwg_finite_difference():
    """d l_aux / d Wg by central differences (routing unchanged by the small step)."""
    rng = np.random.default_rng(2)
    T, H, E, coef = 30, 8, 5, 0.1
    x = rng.normal(size=(T, H))
    wg = rng.normal(size=(H, E)) / np.sqrt(H)
    r = O.route(x, wg, T)
    g = x.T @ O.aux_loss_dlogits(r.expert, r.s, coef)
    eps = 1e-6
    for (h, e) in [(0, 0), (3, 2), (7, 4), (5, 1)]:
        wp, wm = wg.copy(), wg.copy()
        wp[h, e] += eps
        wm[h, e] -= eps
        rp, rm = O.route(x, wp, T), O.route(x, wm, T)
        assert (rp.expert == r.expert).all() and (rm.expert == r.expert).all()
        fd = (O.aux_loss(rp.expert, rp.s, coef) - O.aux_loss(rm.expert, rm.s, coef)) / (2 * eps)
        assert fd == pytest.approx(g[h, e], rel=1e-6, abs=1e-11)
