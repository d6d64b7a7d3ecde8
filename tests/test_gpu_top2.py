"""Top-2 gating (moe_config.top_k = 2, reading R22, NEXT #4) through the C ABI vs
oracle/top2_oracle.py: routing pairs bit-exact outside logged ties, slots and
counts bit-exact after the tie override, outputs and gradients within 1e-2."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from oracle import top2_oracle as T2
from paper_2305_13525_b200 import (MOE_F_AUX_LOSS, MOE_F_RANDOM_PRIORITY, MOE_F_STATS, MoEConfig,
                                   MoELayer, synth)
from tests.helpers import REL_L2_BAR, Inputs, bf16_tensor, rel_l2, tensor_f64

pytestmark = pytest.mark.gpu


def run(inp: Inputs, shape, cf, flags=0, seed=None, coef=0.0):
    cfg = MoEConfig(inp.T, shape.hidden, shape.ffn, shape.experts, cf, 1, 1, True, MOE_F_STATS | flags, coef,
                    top_k=2)
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
    st = layer.moe_stats()
    out = {"y": tensor_f64(y), "dx": tensor_f64(dx), "dwg": dwg.cpu().numpy().astype(np.float64),
           "dw1": tensor_f64(dw1), "dw2": tensor_f64(dw2), "aux": aux, "stats": st,
           **{k: v.cpu().numpy() for k, v in rt.items()}}
    layer.close()
    return out


def check(inp, g, cf, seed=None, coef=0.0):
    xs, dys, wg, w1, w2 = inp.oracle_arrays()
    cap = T2.capacity_top2(inp.T, wg.shape[1], cf)
    order = None if seed is None else O.priority_order(inp.T, seed)
    r0 = T2.route_top2(xs[0], wg, cap, order=order)
    tie = (r0.gap < O.TIE_GAP) | (g["gap"] < O.TIE_GAP)
    bad = np.nonzero((g["expert"] != r0.experts).any(axis=1) & ~tie)[0]
    assert bad.size == 0, f"top-2 routing mismatch outside ties at {bad[:8]}"
    idx = np.nonzero(tie)[0]
    ref = T2.layer_top2(xs, dys, wg, w1, w2, cf, overrides=[(idx, g["expert"][idx])], order=order,
                        aux_coef=coef)
    r = ref["routing"][0]
    np.testing.assert_array_equal(g["slot"], r.slot)
    np.testing.assert_array_equal(g["count"], r.count)
    np.testing.assert_allclose(g["prob"], r.w, rtol=1e-5, atol=1e-6)
    assert g["stats"]["dropped_tokens"] == int((~r.kept).sum())
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
    return r, errs


@pytest.mark.parametrize("cf", [0.5, 1.0, 2.0])
def test_top2_tiny(cf):
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape, skew=1.5)
    r, _ = check(inp, run(inp, shape, cf), cf)
    if cf <= 1.0:
        assert (~r.kept).any()


@pytest.mark.parametrize("T,H,F,E", [(1000, 128, 192, 5), (2048, 256, 512, 16), (3000, 320, 640, 32),
                                     (777, 64, 128, 64), (64, 64, 64, 2), (700, 4096, 128, 16),
                                     (500, 2560, 128, 32)])
def test_top2_ragged(T, H, F, E):
    shape = synth.LayerShape("top2", T, H, F, E)
    inp = Inputs(shape)
    check(inp, run(inp, shape, 1.0), 1.0)


def test_top2_13b_reduced():
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape, tokens=2048)
    check(inp, run(inp, shape, 1.0), 1.0)


def test_top2_with_random_priority_and_aux():
    shape = synth.LayerShape("top2v", 2048, 256, 512, 16)
    inp = Inputs(shape, skew=1.5)
    g = run(inp, shape, 1.0, MOE_F_RANDOM_PRIORITY | MOE_F_AUX_LOSS, seed=31, coef=0.02)
    check(inp, g, 1.0, seed=31, coef=0.02)


def test_top2_exact_ties():
    shape = synth.LayerShape("tie2", 512, 128, 256, 8)
    inp = Inputs(shape)
    inp.wg[:, 5] = inp.wg[:, 2]  # experts 2 and 5 tie everywhere
    g = run(inp, shape, 1.0)
    both = (g["expert"] == 2).any(axis=1) & (g["expert"] == 5).any(axis=1)
    one = (g["expert"] == 2).any(axis=1) ^ (g["expert"] == 5).any(axis=1)
    assert both.any() and not ((g["expert"][:, 0] == 5) & (g["expert"][:, 1] == 2)).any()
    assert not (one & (g["expert"] == 5).any(axis=1)).any()  # lowest index wins a single tie slot
    check(inp, g, 1.0)
