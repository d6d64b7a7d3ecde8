"""NEXT #4 gating variants through the C ABI vs the CPU oracle (1 GPU):
random token-selection priority (MOE_F_RANDOM_PRIORITY, reading R20) — slots,
counts and dropped sets bit-exact — and the auxiliary load-balancing loss
(MOE_F_AUX_LOSS, reading R21) — l_aux and the gate gradients it adds."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2305_13525_b200 import (MOE_F_AUX_LOSS, MOE_F_RANDOM_PRIORITY, MOE_F_STATS, MoEConfig,
                                   MoEError, MoELayer, synth)
from tests.helpers import REL_L2_BAR, Inputs, bf16_tensor, rel_l2, routing_protocol, tensor_f64

pytestmark = pytest.mark.gpu


def run(inp: Inputs, shape, flags, seed=None, coef=0.0, cf=None):
    cfg = MoEConfig(inp.T, shape.hidden, shape.ffn, shape.experts, shape.cf if cf is None else cf, 1, 1, True,
                    MOE_F_STATS | flags, coef)
    layer = MoELayer(cfg)
    if seed is not None:
        layer.moe_set_priority_seed(seed)
    x, dy = bf16_tensor(inp.x[0]), bf16_tensor(inp.dy[0])
    wg = torch.from_numpy(inp.wg).cuda()
    w1, w2 = bf16_tensor(inp.w1), bf16_tensor(inp.w2)
    y, saved = layer.moe_forward(x, wg, w1, w2)
    dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wg, w1, w2)
    rt = layer.moe_routing(saved)
    aux = layer.moe_aux_loss(saved).item() if flags & MOE_F_AUX_LOSS else None
    torch.cuda.synchronize()
    out = {"y": tensor_f64(y), "dx": tensor_f64(dx), "dwg": dwg.cpu().numpy().astype(np.float64),
           "dw1": tensor_f64(dw1), "dw2": tensor_f64(dw2), "aux": aux,
           **{k: v.cpu().numpy() for k, v in rt.items()}}
    layer.close()
    return out


def check(inp, g, cf, seed=None, coef=0.0):
    xs, dys, wg, w1, w2 = inp.oracle_arrays()
    cap = O.capacity(inp.T, wg.shape[1], cf, 1)
    order = None if seed is None else O.priority_order(inp.T, seed)
    r0 = O.route(xs[0], wg, cap, order=order)
    idx, ex = routing_protocol(g["expert"], g["gap"], r0)
    ref = O.layer(xs, dys, wg, w1, w2, cf, 1, overrides=[(idx, ex)], priority_seed=seed, aux_coef=coef)
    r = ref["routing"][0]
    np.testing.assert_array_equal(g["slot"], r.slot)
    np.testing.assert_array_equal(g["count"], r.count)
    errs = {"y": rel_l2(g["y"], ref["y"][0]), "dx": rel_l2(g["dx"], ref["dx"][0]),
            "dwg": rel_l2(g["dwg"], ref["dwg"][0]), "dw1": rel_l2(g["dw1"], ref["dw1"]),
            "dw2": rel_l2(g["dw2"], ref["dw2"])}
    for k, v in errs.items():
        assert v <= REL_L2_BAR, (k, errs)
    from tests.helpers import parity_failures
    rows = []
    for k in ("y", "dx", "dw1", "dw2"):
        want = ref[k][0] if k in ("y", "dx") else ref[k]
        rows += parity_failures(k, g[k], want)
    assert not rows, rows
    if coef:
        assert g["aux"] == pytest.approx(ref["aux"][0], rel=1e-5)
    return r, ref


@pytest.mark.parametrize("seed", [0, 7, (1 << 40) + 3])
@pytest.mark.parametrize("cf", [0.5, 1.0])
def test_random_priority_tiny(seed, cf):
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape, skew=1.5)
    g = run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=seed, cf=cf)
    r, _ = check(inp, g, cf, seed=seed)
    assert (~r.kept).any()


@pytest.mark.parametrize("T,H,F,E", [(1000, 128, 192, 5), (3000, 320, 640, 32), (777, 64, 128, 64)])
def test_random_priority_ragged(T, H, F, E):
    shape = synth.LayerShape("rts", T, H, F, E)
    inp = Inputs(shape, skew=1.3)
    check(inp, run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=T), 1.0, seed=T)


def test_random_priority_13b_reduced():
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape, tokens=2048, skew=1.5)
    check(inp, run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=99), 1.0, seed=99)


def test_random_priority_full_size_slots():
    """T = 16384 (the bench's configuration): the slot assignment, bit-exact."""
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape, skew=1.5)
    g = run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=123)
    xs, _, wg, _, _ = inp.oracle_arrays()
    cap = O.capacity(inp.T, shape.experts, 1.0)
    order = O.priority_order(inp.T, 123)
    r0 = O.route(xs[0], wg, cap, order=order)
    idx, ex = routing_protocol(g["expert"], g["gap"], r0)
    r = O.route(xs[0], wg, cap, override=(idx, ex), order=order)
    np.testing.assert_array_equal(g["slot"], r.slot)
    np.testing.assert_array_equal(g["count"], r.count)


def test_random_priority_seed_changes_slots_only():
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape, skew=1.5)
    a = run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=1)
    b = run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=2)
    c = run(inp, shape, MOE_F_RANDOM_PRIORITY, seed=1)
    np.testing.assert_array_equal(a["expert"], b["expert"])
    assert not np.array_equal(a["slot"], b["slot"])
    for k in ("y", "dx", "dwg", "dw1", "dw2", "slot"):
        np.testing.assert_array_equal(a[k], c[k])


@pytest.mark.parametrize("coef", [0.01, 1.0])
def test_aux_loss_tiny(coef):
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape, skew=1.5)
    g = run(inp, shape, MOE_F_AUX_LOSS, coef=coef)
    r, ref = check(inp, g, 1.0, coef=coef)
    assert (~r.kept).any()
    assert np.abs(g["dx"][~r.kept]).max() > 0  # dropped tokens get the aux gate gradient


@pytest.mark.parametrize("T,H,F,E", [(1000, 128, 192, 5), (2048, 256, 512, 16), (777, 64, 128, 64)])
def test_aux_loss_ragged(T, H, F, E):
    shape = synth.LayerShape("aux", T, H, F, E)
    inp = Inputs(shape, skew=1.3)
    check(inp, run(inp, shape, MOE_F_AUX_LOSS, coef=0.1), 1.0, coef=0.1)


def test_aux_and_random_priority_13b_reduced():
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape, tokens=2048, skew=1.5)
    flags = MOE_F_AUX_LOSS | MOE_F_RANDOM_PRIORITY
    check(inp, run(inp, shape, flags, seed=5, coef=0.05), 1.0, seed=5, coef=0.05)


def test_aux_loss_needs_flag():
    shape = synth.CONFIGS["tiny"]
    layer = MoELayer(MoEConfig.from_shape(shape))
    saved = layer.new_saved()
    with pytest.raises(MoEError) as ei:
        layer.moe_aux_loss(saved)
    assert ei.value.name == "MOE_ERR_STATE"
    layer.close()
