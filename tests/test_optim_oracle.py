"""Pins of oracle/optim_oracle.py (the tiled optimizer)
against things other than itself: the tile-plan and memory law the paper
states, closed forms of Adam's bias correction, the
zero-gradient special case, and torch.optim.AdamW (a library routine) — plus
the C ABI's plan / validation entry points (no GPU compute)."""
import math

import numpy as np
import pytest
import torch

from oracle import optim_oracle as OO
from paper_2305_13525_b200 import MoEError, moe_adamw_plan, moe_adamw_step


def _state(n, seed=0):
    rng = np.random.default_rng(seed)
    g = rng.normal(0, 1e-2, n).astype(np.float32)
    gbits = OO.bf16_round_bits(g)
    p = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = np.abs(rng.normal(0, 1e-5, n)).astype(np.float32)
    return gbits, p, m, v


def _g32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------- tile plan / memory law
def test_tile_plan_examples():
    assert OO.tile_plan(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert OO.tile_plan(10, 10) == [(0, 10)]
    assert OO.tile_plan(0, 4) == []
    with pytest.raises(ValueError):
        OO.tile_plan(10, 0)


@pytest.mark.parametrize("n,ts", [(1, 1), (10, 3), (4096, 1000), (1000, 4096), (12345, 1)])
def test_tile_plan_covers_disjoint(n, ts):
    plan = OO.tile_plan(n, ts)
    assert len(plan) == -(-n // ts)
    assert plan[0][0] == 0 and plan[-1][1] == n
    for (a, b), (c, _) in zip(plan, plan[1:]):
        assert b == c and b - a == ts
    assert all(0 < b - a <= ts for a, b in plan)


def test_transient_memory_law():
    """4 x ts bytes tiled (independent of n), 4 x n untiled."""
    for n in (1000, 5000, 20000):
        gb, p, m, v = _state(n)
        h = OO.AdamW(step=3)
        assert OO.adamw_untiled(gb, p, m, v, h)[4] == 4 * n
        assert OO.adamw_tiled(gb, p, m, v, h, 1000)[4] == 4000
    gb, p, m, v = _state(300)
    assert OO.adamw_tiled(gb, p, m, v, OO.AdamW(), 1000)[4] == 1200  # ts > n: one short tile


def test_paper_tile_size():
    assert OO.TILE_PARAMS_PAPER == 1_800_000
    # "caps the spike in the optimizer step to 1 GB"? 4 B x 1.8 M = 7.2 MB per buffer; the paper's
    # 1 GB figure is the whole optimizer step's spike, not the gradient buffer — only the 4 x ts law is pinned.
    assert 4 * OO.TILE_PARAMS_PAPER == 7_200_000


# ---------------------------------------------------------------- tiled == untiled
def test_tiled_equals_untiled_exhaustive_small():
    n = 37
    gb, p, m, v = _state(n, 1)
    h = OO.AdamW(step=5)
    ref = OO.adamw_untiled(gb, p, m, v, h)
    for ts in range(1, n + 2):
        out = OO.adamw_tiled(gb, p, m, v, h, ts)
        for a, b in zip(ref[:4], out[:4]):
            np.testing.assert_array_equal(a, b)


def test_tiled_equals_untiled_random():
    gb, p, m, v = _state(4096, 42)
    h = OO.AdamW(step=7)
    ref = OO.adamw_untiled(gb, p, m, v, h)
    out = OO.adamw_tiled(gb, p, m, v, h, 1000)
    for a, b in zip(ref[:4], out[:4]):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- the update rule
def test_zero_gradient_zero_moments_is_pure_decay():
    n = 257
    _, p, _, _ = _state(n)
    z = np.zeros(n, np.float32)
    h = OO.AdamW(lr=1e-3, weight_decay=0.1, step=4)
    p2, m2, v2, _, _ = OO.adamw_untiled(np.zeros(n, np.uint16), p, z, z, h)
    np.testing.assert_array_equal(m2, 0)
    np.testing.assert_array_equal(v2, 0)
    np.testing.assert_array_equal(p2, p * np.float32(1 - 1e-3 * 0.1))


def test_first_step_closed_form():
    """t = 1, m = v = 0: m_hat = g, sqrt(v_hat) = |g| -> p' = p (1 - lr wd) - lr g / (|g| + eps)."""
    n = 2000
    gb, p, _, _ = _state(n, 3)
    z = np.zeros(n, np.float32)
    h = OO.AdamW(lr=1e-3, weight_decay=0.05, step=1, eps=1e-8)
    p2 = OO.adamw_untiled(gb, p, z, z, h)[0].astype(np.float64)
    g = _g32(gb).astype(np.float64)
    want = p.astype(np.float64) * (1 - 1e-3 * 0.05) - 1e-3 * g / (np.abs(g) + 1e-8)
    np.testing.assert_allclose(p2, want, rtol=4e-7, atol=1e-10)  # a few binary32 ulps


def test_constant_gradient_bias_correction():
    """k steps of a constant gradient from m = v = 0: m_k = (1 - b1^k) g, v_k = (1 - b2^k) g^2,
    so the bias-corrected step is lr g / (|g| + eps) every time."""
    n = 500
    gb, p0, _, _ = _state(n, 5)
    g = _g32(gb).astype(np.float64)
    p, m, v = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    lr, wd, b1, b2 = 1e-3, 0.0, 0.9, 0.95
    want = p0.astype(np.float64)
    for k in range(1, 6):
        p, m, v, _, _ = OO.adamw_untiled(gb, p, m, v, OO.AdamW(lr=lr, beta1=b1, beta2=b2, weight_decay=wd, step=k))
        want = want - lr * g / (np.abs(g) + 1e-8)
        np.testing.assert_allclose(m, (1 - b1 ** k) * g, rtol=1e-5, atol=1e-12)
        np.testing.assert_allclose(v, (1 - b2 ** k) * g * g, rtol=1e-5, atol=1e-16)
    np.testing.assert_allclose(p, want, rtol=1e-6, atol=2e-9)  # 5 steps of 1e-3: ~1e-6 relative to the motion


def test_matches_torch_adamw():
    """Library routine: torch.optim.AdamW (single-tensor, fp32 CPU) over 4 steps."""
    n = 3000
    rng = np.random.default_rng(11)
    p0 = rng.normal(0, 0.02, n).astype(np.float32)
    grads = [OO.bf16_round_bits(rng.normal(0, 1e-2, n).astype(np.float32)) for _ in range(4)]
    hp = dict(lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    t = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.AdamW([t], lr=hp["lr"], betas=(hp["beta1"], hp["beta2"]), eps=hp["eps"],
                            weight_decay=hp["weight_decay"], foreach=False, fused=False)
    p, m, v = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for k, gb in enumerate(grads, start=1):
        t.grad = torch.from_numpy(_g32(gb).copy())
        opt.step()
        p, m, v, _, _ = OO.adamw_untiled(gb, p, m, v, OO.AdamW(step=k, **hp))
    st = opt.state[t]
    np.testing.assert_allclose(p, t.detach().numpy(), rtol=0, atol=1e-7)
    np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-5, atol=1e-12)


def test_bf16_copy_is_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e-3], np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(OO.bf16_round_bits(x), want)


def test_host_scalars():
    s = OO.host_scalars(OO.AdamW(lr=1e-3, beta1=0.9, beta2=0.99, step=2, weight_decay=0.1))
    assert s["step"] == np.float32(1e-3 / (1 - 0.81))
    assert s["c2s"] == np.float32(math.sqrt(1 - 0.99 ** 2))
    assert s["decay"] == np.float32(1 - 1e-4)
    with pytest.raises(ValueError):
        OO.host_scalars(OO.AdamW(step=0))


# ---------------------------------------------------------------- C ABI (no GPU compute)
def test_abi_plan():
    assert moe_adamw_plan(10, 4) == (3, 16)
    assert moe_adamw_plan(10, 10) == (1, 40)
    assert moe_adamw_plan(0, 4) == (0, 0)
    assert moe_adamw_plan(10, 0) == (1, 0)  # fused: no temporary
    assert moe_adamw_plan(537_919_488, OO.TILE_PARAMS_PAPER) == (299, 7_200_000)
    with pytest.raises(MoEError):
        moe_adamw_plan(-1, 4)


class _NullStream:
    cuda_stream = 0


def test_abi_step_validation():
    """Rejected before anything is enqueued (host pointers never dereferenced)."""
    x = torch.zeros(16)
    kw = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0, stream=_NullStream())
    with pytest.raises(MoEError) as ei:  # step 0
        moe_adamw_step(x, x, x, x, step=0, **kw)
    assert ei.value.name == "MOE_ERR_ARG"
    with pytest.raises(MoEError) as ei:  # tiled without temp
        moe_adamw_step(x, x, x, x, step=1, tile_params=4, **kw)
    assert ei.value.name == "MOE_ERR_ARG"
    with pytest.raises(MoEError) as ei:  # fused with temp
        moe_adamw_step(x, x, x, x, step=1, temp=x, **kw)
    assert ei.value.name == "MOE_ERR_ARG"
    with pytest.raises(MoEError) as ei:  # misaligned
        moe_adamw_step(x[1:], x[1:], x[1:], x[1:], step=1, **kw)
    assert ei.value.name == "MOE_ERR_ALIGN"
