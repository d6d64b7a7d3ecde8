"""MoE layer (1 GPU, G = 1) through the C ABI vs the CPU oracle.

Routing: bit-exact outside logged ties (BASELINE.json); slots/count/dropped
sets bit-exact after the tie-override protocol.
Floating outputs: relative L2 <= 1e-2 for y, dx, dWg, dW1, dW2.
"""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2305_13525_b200 import MoEConfig, MoELayer, synth
from tests.helpers import REL_L2_BAR, Inputs, bf16_tensor, rel_l2, routing_protocol, tensor_f64

pytestmark = pytest.mark.gpu


def run_gpu(inp: Inputs, shape, forced=None, cf=None):
    cfg = MoEConfig(inp.T, shape.hidden, shape.ffn, shape.experts,
                    shape.cf if cf is None else cf, 1, 1, True, 1 | (2 if forced is not None else 0))
    layer = MoELayer(cfg)
    x = bf16_tensor(inp.x[0])
    dy = bf16_tensor(inp.dy[0])
    wg = torch.from_numpy(inp.wg).cuda()
    w1 = bf16_tensor(inp.w1)
    w2 = bf16_tensor(inp.w2)
    f = None if forced is None else torch.from_numpy(forced).cuda()
    y, saved = layer.moe_forward(x, wg, w1, w2, forced=f)
    dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wg, w1, w2)
    rt = layer.moe_routing(saved)
    torch.cuda.synchronize()
    out = {"y": tensor_f64(y), "dx": tensor_f64(dx), "dwg": dwg.cpu().numpy().astype(np.float64),
           "dw1": tensor_f64(dw1), "dw2": tensor_f64(dw2),
           **{k: v.cpu().numpy() for k, v in rt.items()}, "stats": layer.moe_stats()}
    layer.close()
    return out, cfg


def check_parity(inp: Inputs, g, cf, forced=None):
    xs, dys, wg, w1, w2 = inp.oracle_arrays()
    cap = O.capacity(inp.T, wg.shape[1], cf, 1)
    r0 = O.route(xs[0], wg, cap, forced=forced)
    if forced is None:
        idx, ex = routing_protocol(g["expert"], g["gap"], r0)
        override = [(idx, ex)]
    else:
        np.testing.assert_array_equal(g["expert"], forced)
        override = None
    ref = O.layer(xs, dys, wg, w1, w2, cf, 1, forced=None if forced is None else [forced],
                  overrides=override)
    r = ref["routing"][0]
    np.testing.assert_array_equal(g["slot"], r.slot)
    np.testing.assert_array_equal(g["count"], r.count)
    np.testing.assert_allclose(g["prob"], r.p, rtol=1e-5, atol=1e-7)
    assert g["stats"]["dropped_tokens"] == int((~r.kept).sum())
    errs = {"y": rel_l2(g["y"], ref["y"][0]), "dx": rel_l2(g["dx"], ref["dx"][0]),
            "dwg": rel_l2(g["dwg"], ref["dwg"][0]), "dw1": rel_l2(g["dw1"], ref["dw1"]),
            "dw2": rel_l2(g["dw2"], ref["dw2"])}
    for k, v in errs.items():
        assert v <= REL_L2_BAR, (k, errs)
    from tests.helpers import parity_failures
    fails = []
    for k, want in (("y", ref["y"][0]), ("dx", ref["dx"][0]), ("dw1", ref["dw1"]), ("dw2", ref["dw2"])):
        fails += parity_failures(k, g[k], want)
    assert not fails, fails
    # dropped tokens are exact zeros
    assert (g["y"][~r.kept] == 0).all() and (g["dx"][~r.kept] == 0).all()
    return errs


@pytest.mark.parametrize("cf", [1.0, 0.5, 2.0])
def test_tiny_layer_parity(cf):
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape)
    g, _ = run_gpu(inp, shape, cf=cf)
    check_parity(inp, g, cf)


def test_tiny_skewed_drops():
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape, skew=1.5)
    g, _ = run_gpu(inp, shape)
    errs = check_parity(inp, g, 1.0)
    assert g["stats"]["dropped_tokens"] > 0, errs


@pytest.mark.parametrize("mode", ["round_robin", "all_to_one", "random"])
def test_tiny_forced_routing(mode):
    shape = synth.CONFIGS["tiny"]
    inp = Inputs(shape)
    forced = synth.forced_routing(mode, inp.T, shape.experts)
    g, _ = run_gpu(inp, shape, forced=forced)
    check_parity(inp, g, 1.0, forced=forced)
    if mode == "round_robin":
        assert g["stats"]["dropped_tokens"] == 0
    if mode == "all_to_one":
        assert g["count"][0] == g["count"].sum() == O.capacity(inp.T, shape.experts, 1.0)


@pytest.mark.parametrize("T,H,F,E", [(1000, 128, 192, 5), (2048, 256, 512, 16), (3000, 320, 640, 32),
                                     (777, 64, 128, 64), (1, 64, 64, 3),
                                     # expert-split gate (Wg > 128 KiB): 6.7B / 2.7B / E = 64 widths
                                     (1000, 4096, 256, 16), (600, 2560, 128, 32), (500, 2048, 128, 64)])
def test_ragged_shapes(T, H, F, E):
    shape = synth.LayerShape("ragged", T, H, F, E)
    inp = Inputs(shape)
    g, _ = run_gpu(inp, shape)
    check_parity(inp, g, 1.0)


def test_exact_tie_lowest_index():
    shape = synth.LayerShape("tie", 512, 128, 256, 8)
    inp = Inputs(shape)
    inp.wg[:, 5] = inp.wg[:, 2]  # exact ties between experts 2 and 5
    g, _ = run_gpu(inp, shape)
    xs, dys, wg, w1, w2 = inp.oracle_arrays()
    r = O.route(xs[0], wg, O.capacity(512, 8, 1.0))
    tied = r.expert == 2
    assert (g["expert"][tied] == 2).all() and not (g["expert"] == 5).any()
    assert g["stats"]["tie_tokens"] >= int(tied.sum())
    check_parity(inp, g, 1.0)


def test_13b_reduced_tokens_full_parity():
    """1.3B shapes (H 2048, F 8192, E 16) at T = 2048, every output element."""
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape, tokens=2048)
    g, _ = run_gpu(inp, shape)
    check_parity(inp, g, 1.0)


def test_13b_full_size_sampled():
    """BASELINE configs[1] at full size (T = 16384) in the bench's launch configuration:
    routing of every token bit-exact; y / dx on one token per (expert, 256-row M-tile) of the
    expert GEMMs (every M-tile of F6/F7/B4/B5 covered) plus dropped tokens; dW1 rows / dW2
    columns on one f per 256-wide tile of every expert (every M-tile of dW1 and N-tile of
    dW2, all H). Global rel L2 <= 1e-2 and <= 5e-2 per sampled row (a single corrupted tile
    cannot hide under the global norm)."""
    from tests.helpers import LazyExperts, parity_failures, stratified_f, stratified_tokens
    shape = synth.CONFIGS["1.3b"]
    inp = Inputs(shape)
    g, _ = run_gpu(inp, shape)
    x = O.decode_bf16(inp.x[0])
    dy = O.decode_bf16(inp.dy[0])
    wg = inp.wg.astype(np.float64)
    w1, w2 = LazyExperts(inp.w1), LazyExperts(inp.w2)
    cap = O.capacity(inp.T, shape.experts, 1.0)
    r0 = O.route(x, wg, cap)
    idx, ex = routing_protocol(g["expert"], g["gap"], r0)
    r = O.route(x, wg, cap, override=(idx, ex))
    np.testing.assert_array_equal(g["slot"], r.slot)
    np.testing.assert_array_equal(g["count"], r.count)
    toks = stratified_tokens(r, 0)
    assert len(toks) >= shape.experts * (cap // 256)
    yr, dxr = O.tokens_forward_backward(toks, x, dy, wg, w1, w2, r)
    fails = parity_failures("y", g["y"][toks], yr) + parity_failures("dx", g["dx"][toks], dxr)
    fl = stratified_f(shape.ffn)
    got1, want1, got2, want2 = [], [], [], []
    for e in range(shape.experts):
        for f in fl:
            a, b = O.expert_row_grads(e, int(f), [x], [dy], w1, w2, [r])
            want1.append(a)
            want2.append(b)
            got1.append(g["dw1"][e, f])
            got2.append(g["dw2"][e, :, f])
    fails += parity_failures("dw1", np.array(got1), np.array(want1))
    fails += parity_failures("dw2", np.array(got2), np.array(want2))
    assert not fails, fails


def test_determinism_bitwise():
    shape = synth.LayerShape("det", 4096, 256, 512, 16)
    inp = Inputs(shape)
    a, _ = run_gpu(inp, shape)
    b, _ = run_gpu(inp, shape)
    for k in ("y", "dx", "dwg", "dw1", "dw2", "slot"):
        np.testing.assert_array_equal(a[k], b[k])


def test_forward_errors_are_status_codes():
    from paper_2305_13525_b200 import MoEError
    shape = synth.CONFIGS["tiny"]
    layer = MoELayer(MoEConfig.from_shape(shape))
    x = torch.zeros(shape.tokens, shape.hidden, dtype=torch.bfloat16, device="cuda")
    wg = torch.zeros(shape.hidden, shape.experts, device="cuda")
    w1 = torch.zeros(shape.experts, shape.ffn, shape.hidden, dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros(shape.experts, shape.hidden, shape.ffn, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(MoEError) as ei:  # forced routing not enabled
        layer.moe_forward(x, wg, w1, w2, forced=torch.zeros(shape.tokens, dtype=torch.int32, device="cuda"))
    assert ei.value.name == "MOE_ERR_ARG"
    bogus = layer.new_saved()
    with pytest.raises(MoEError) as ei:  # saved blob never written by moe_forward
        layer.moe_backward(x, bogus, x, wg, w1, w2)
    assert ei.value.name == "MOE_ERR_STATE"
    # x = 0: every token routes to expert 0 with p = 1/E (oracle special case)
    y, saved = layer.moe_forward(x, wg, w1, w2)
    rt = layer.moe_routing(saved)
    assert (rt["expert"] == 0).all() and torch.allclose(rt["prob"], torch.full_like(rt["prob"], 0.25))
    layer.close()


@pytest.mark.parametrize("cac", [True, False])
def test_checkpoint_replay_bitwise(cac):
    """Checkpointed forward + replay + backward == plain forward + backward, bitwise."""
    from paper_2305_13525_b200 import MOE_F_CAC, MOE_F_CHECKPOINT, MoEError
    shape = synth.LayerShape("ck", 2048, 256, 512, 8)
    inp = Inputs(shape)
    x, dy = bf16_tensor(inp.x[0]), bf16_tensor(inp.dy[0])
    wg = torch.from_numpy(inp.wg).cuda()
    w1, w2 = bf16_tensor(inp.w1), bf16_tensor(inp.w2)
    base = MoEConfig.from_shape(shape)
    outs = []
    for flags in (base.flags, base.flags | MOE_F_CHECKPOINT | (MOE_F_CAC if cac else 0)):
        layer = MoELayer(MoEConfig(shape.tokens, shape.hidden, shape.ffn, shape.experts, 1.0, 1, 1, True, flags))
        y, saved = layer.moe_forward(x, wg, w1, w2)
        if flags & MOE_F_CHECKPOINT:
            with pytest.raises(MoEError) as ei:
                layer.moe_backward(dy, saved, x, wg, w1, w2)
            assert ei.value.name == "MOE_ERR_STATE"
            layer.moe_forward_replay(saved, x, wg, w1, w2)
        g = layer.moe_backward(dy, saved, x, wg, w1, w2)
        rt = layer.moe_routing(saved)
        torch.cuda.synchronize()
        outs.append((y.clone(), *[t.clone() for t in g]))
        st = layer.moe_stats()
        layer.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # the checkpointed path itself against the oracle (the replay must
    # reproduce the forward's activations, not merely agree with another GPU run)
    names = ("y", "dx", "dwg", "dw1", "dw2")
    gck = {k: (tensor_f64(v) if v.dtype == torch.bfloat16 else v.cpu().numpy().astype(np.float64))
           for k, v in zip(names, outs[1])}
    gck.update({k: v.cpu().numpy() for k, v in rt.items()})
    gck["stats"] = st
    check_parity(inp, gck, 1.0)


def test_fused_gate_dx_matches_separate_kernel(monkeypatch):
    """B5's gate-dx epilogue (one GPU, top-1) vs the separate B10 kernel (MOE_NO_FUSED_DX=1):
    y and the expert gradients bitwise, dx / dWg to rounding (the fused path adds the gate
    term before the bf16 rounding of the B5 accumulator)."""
    shape = synth.LayerShape("fdx", 4096, 256, 512, 16)
    inp = Inputs(shape, skew=1.3)
    monkeypatch.setenv("MOE_NO_FUSED_DX", "0")
    a, _ = run_gpu(inp, shape)
    monkeypatch.setenv("MOE_NO_FUSED_DX", "1")
    b, _ = run_gpu(inp, shape)
    for k in ("y", "dw1", "dw2", "slot"):
        np.testing.assert_array_equal(a[k], b[k])
    assert rel_l2(a["dx"], b["dx"]) < 3e-3 and rel_l2(a["dwg"], b["dwg"]) < 1e-5
    check_parity(inp, a, 1.0)


def test_fused_combine_matches_separate_kernel(monkeypatch):
    """F7's combine epilogue (one GPU, top-1) vs the separate F11 kernel
    (MOE_NO_FUSED_COMBINE=1): every gradient bitwise (O is stored the same way), y to
    rounding (the fused path scales the fp32 accumulator before the bf16 rounding)."""
    shape = synth.LayerShape("fcb", 4096, 256, 512, 16)
    inp = Inputs(shape, skew=1.3)
    monkeypatch.setenv("MOE_NO_FUSED_COMBINE", "0")
    a, _ = run_gpu(inp, shape)
    monkeypatch.setenv("MOE_NO_FUSED_COMBINE", "1")
    b, _ = run_gpu(inp, shape)
    for k in ("dx", "dwg", "dw1", "dw2", "slot"):
        np.testing.assert_array_equal(a[k], b[k])
    assert rel_l2(a["y"], b["y"]) < 3e-3
    check_parity(inp, a, 1.0)


@pytest.mark.parametrize("T,H,E", [(16384, 2048, 16), (4096, 4096, 16), (4096, 2560, 32), (3000, 2048, 64),
                                   (1000, 128, 5)])
def test_gate_logit_error(T, H, E):
    """F1 on the tensor cores (Wg split hi + mid + lo, a fresh TMEM accumulator per 64-wide
    k block, Kahan sum of the blocks): the saved logits (first region of the saved blob,
    plan.cpp make_layouts) against the float64 x . Wg of the oracle: rms <= 1.5e-7 and
    max <= 8e-7 (measured rms 7.8e-8, max 4-6e-7 over 4k-262k logits, about what a
    pairwise fp32 sum gives; a sequential fp32 sum of 2048 terms has ~8e-7 rms). Routing
    outside the logged ties (gap < 1e-6, BASELINE.json) is checked by the layer tests and
    test_gate_near_ties."""
    shape = synth.LayerShape("gate", T, H, 256, E)
    x_bits = synth.make_x(shape)
    wg = synth.make_wg(shape)
    cfg = MoEConfig(T, H, 256, E, 1.0, 1, 1, True, 1)
    layer = MoELayer(cfg)
    x = bf16_tensor(x_bits)
    w1 = torch.zeros((E, 256, H), dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros((E, H, 256), dtype=torch.bfloat16, device="cuda")
    y, saved = layer.moe_forward(x, torch.from_numpy(wg).cuda(), w1, w2)
    torch.cuda.synchronize()
    got = saved[: T * E * 4].view(torch.float32).reshape(T, E).cpu().numpy().astype(np.float64)
    layer.close()
    ref = O.decode_bf16(x_bits) @ wg.astype(np.float64)
    err = np.abs(got - ref)
    srt = np.sort(ref, axis=1)
    gap = srt[:, -1] - srt[:, -2] if E > 1 else np.full(T, np.inf)
    near = gap < 1e-5
    near_err = err[near].max() if near.any() else 0.0
    print(f"gate logit error T={T} H={H} E={E}: max {err.max():.3e}, rms {np.sqrt(np.mean(err ** 2)):.3e}, "
          f"{int(near.sum())} near-tie tokens max {near_err:.3e}")
    assert np.sqrt(np.mean(err ** 2)) <= 1.5e-7 and err.max() <= 8e-7, err.max()


def test_gate_near_ties():
    """Many near ties: expert 1's gate column is expert 0's plus a tiny perturbation, so
    a large share of tokens has a top-2 gap of ~1e-6 .. 1e-5; routing must still match the
    oracle outside the logged (< 1e-6) ties."""
    T, H, E = 4096, 2048, 8
    shape = synth.LayerShape("ties", T, H, 256, E)
    x_bits = synth.make_x(shape)
    wg = synth.make_wg(shape)
    rng = np.random.default_rng(5)
    wg[:, 0] = np.abs(wg[:, 0]) * 4.0  # expert 0 wins clearly ...
    wg[:, 1] = wg[:, 0] + (rng.standard_normal(H) * 2e-7).astype(np.float32)  # ... unless expert 1 is nearer
    cfg = MoEConfig(T, H, 256, E, 8.0, 1, 1, True, 1)
    layer = MoELayer(cfg)
    x = bf16_tensor(x_bits)
    w1 = torch.zeros((E, 256, H), dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros((E, H, 256), dtype=torch.bfloat16, device="cuda")
    y, saved = layer.moe_forward(x, torch.from_numpy(wg).cuda(), w1, w2)
    rt = layer.moe_routing(saved)
    torch.cuda.synchronize()
    ge, gg = rt["expert"].cpu().numpy(), rt["gap"].cpu().numpy()
    layer.close()
    r0 = O.route(O.decode_bf16(x_bits), wg.astype(np.float64), O.capacity(T, E, 8.0))
    tie = (r0.gap < O.TIE_GAP) | (gg < O.TIE_GAP)
    near = r0.gap < 1e-5
    assert near.sum() > T // 4, int(near.sum())  # the case really is near-tie heavy
    bad = np.nonzero((ge != r0.expert) & ~tie)[0]
    assert bad.size == 0, (bad[:10], r0.gap[bad[:10]])
