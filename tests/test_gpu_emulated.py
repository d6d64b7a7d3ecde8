"""The 10 exchange rows (F4, F5, F8, F9, F10, B2, B3, B7, B8, B9) on ONE GPU, vs the oracle.

Every rank of a (G_t, G_ep) layout runs in this process as an emulated rank (tests/emu.py,
include/moe.h moe_emu_group): the product kernels of the multi-GPU path — fused peer
dispatch with DTD's folded all-gather, the split copy-engine
all-to-all (G_t = 1), the fused TP reduction + return exchange (reduce-scatter under DTD,
all-reduce under vanilla), the combine-backward peer stores —
with only the window publication replaced by stream-ordered events. Compared with the CPU
oracle over all token groups; DTD == vanilla bitwise at G_t <= 2; the a2a ledger of
vanilla is G_t x DTD's; CAC / plain checkpoint replays are bitwise.
"""
import numpy as np
import pytest
import torch

from paper_2305_13525_b200 import (MOE_F_NVLS, MOE_F_AUX_LOSS, MOE_F_CAC, MOE_F_CHECKPOINT, MOE_F_RANDOM_PRIORITY,
                                   EmuGroup, MoEComm, MoEError, MoELayer, moe_comm_plan_bytes,
                                   moe_plan_collectives, synth)
from tests import emu

pytestmark = pytest.mark.gpu

LAYOUTS = [(2, 1), (1, 2), (2, 2), (4, 1), (1, 4), (2, 4), (1, 8), (4, 2)]  # (G_t, G_ep), world = G_t*G_ep


def _shape(gt, gep, T=512, H=256, F=512, cf=1.0):
    return synth.LayerShape(f"emu-tp{gt}ep{gep}", T, H, F, max(8, 2 * gep), cf, gt, gep)


def _ledger(st, cfg, world, rank):
    plan = moe_plan_collectives(cfg, world, rank)
    want = {}
    for c in plan:
        want[c["kind"]] = want.get(c["kind"], 0) + c["wire_bytes"]
    got = {k: v for k, v in st["wire_bytes"].items() if v}
    return [] if got == want else [f"rank {rank}: ledger {got} != plan {want}"]


@pytest.mark.parametrize("gt,gep", LAYOUTS)
def test_emulated_exchange_parity(gt, gep):
    wl = emu.Workload(_shape(gt, gep))
    modes = {"dtd": wl.config(True), "van": wl.config(False),
             "cac": wl.config(True, MOE_F_CHECKPOINT | MOE_F_CAC), "ckpt": wl.config(True, MOE_F_CHECKPOINT)}
    if gt > 1:  # the NVLS data flow (own-slice a2a, then a TP-group all-gather), unicast-emulated
        modes["nvls"] = wl.config(True, MOE_F_NVLS)
    res = emu.run_modes(wl, modes, replay_keys=("cac", "ckpt"))
    if gt > 1:
        fails_nv = emu.bitwise_failures(res, "dtd", "nvls")
        for r, rr in enumerate(res):
            fails_nv += _ledger(rr["nvls"]["stats"], modes["nvls"], wl.world, r)
            ag_f, ag_n = rr["dtd"]["stats"]["wire_bytes"]["allgather"], rr["nvls"]["stats"]["wire_bytes"]["allgather"]
            if ag_n * (gt - 1) != ag_f:
                fails_nv.append(f"rank {r}: NVLS all-gather egress {ag_n} x {gt - 1} != folded {ag_f}")
        assert not fails_nv, "\n".join(fails_nv[:40])
    fails, errs = emu.oracle_failures(wl, res, "dtd")
    fails += emu.oracle_failures(wl, res, "van")[0]
    fails += (emu.bitwise_failures if gt <= 2 else emu.close_failures)(res, "dtd", "van")
    fails += emu.bitwise_failures(res, "dtd", "cac") + emu.bitwise_failures(res, "dtd", "ckpt")
    for r, rr in enumerate(res):
        fails += _ledger(rr["dtd"]["stats"], modes["dtd"], wl.world, r)
        fails += _ledger(rr["van"]["stats"], modes["van"], wl.world, r)
        a2a_d, a2a_v = rr["dtd"]["stats"]["wire_bytes"]["a2a"], rr["van"]["stats"]["wire_bytes"]["a2a"]
        if a2a_d * gt != a2a_v:
            fails.append(f"rank {r}: a2a bytes dtd {a2a_d} x {gt} != vanilla {a2a_v}")
        if rr["cac"]["stats"]["replay_calls"] != 0:
            fails.append(f"rank {r}: CAC replay issued collectives")
        if rr["ckpt"]["stats"]["replay_calls"] != rr["dtd"]["stats"]["forward_calls"]:
            fails.append(f"rank {r}: plain checkpoint replay did not repeat the forward's collectives")
    assert not fails, "\n".join(fails[:40])
    print("max rel L2", {k: max(v for (r, n), v in errs.items() if n == k) for k in ("y", "dx", "dwg", "dw1", "dw2")})


@pytest.mark.parametrize("gep", [2, 4])
def test_emulated_return_paths_bitwise(gep, monkeypatch):
    """G_t = 1 split exchange: the return all-to-all fused into the GEMM epilogues (F7+F9,
    B5+B8 peer stores, the default) against the copy-engine return driven by GEMM2's
    completion flags (MOE_NO_FUSED_RETURN=1) and against the per-part launches
    (+ MOE_NO_GEMM_SIGNAL=1): where rows travel never changes their arithmetic, so all three
    are bitwise equal, and the fused one matches the oracle."""
    wl = emu.Workload(_shape(1, gep))
    fused = emu.run_modes(wl, {"m": wl.config(True)})
    fails = emu.oracle_failures(wl, fused, "m")[0]
    monkeypatch.setenv("MOE_NO_FUSED_RETURN", "1")
    ce = emu.run_modes(wl, {"m": wl.config(True)})
    monkeypatch.setenv("MOE_NO_GEMM_SIGNAL", "1")
    parts = emu.run_modes(wl, {"m": wl.config(True)})
    for other in (ce, parts):
        fails += emu.bitwise_failures([{"a": a["m"], "b": b["m"]} for a, b in zip(fused, other)], "a", "b")
    assert not fails, "\n".join(fails[:40])


@pytest.mark.parametrize("gt,gep", [(2, 2), (4, 1), (1, 4), (2, 4)])
def test_emulated_drops(gt, gep):
    """cf 0.5 with an oversubscribed expert: DTD slices of partly empty capacity buffers."""
    wl = emu.Workload(_shape(gt, gep, T=600, cf=0.5), skew=1.5)
    modes = {"dtd": wl.config(True), "van": wl.config(False)}
    res = emu.run_modes(wl, modes)
    assert any(rr["dtd"]["stats"]["dropped_tokens"] > 0 for rr in res)
    fails = emu.oracle_failures(wl, res, "dtd")[0] + emu.oracle_failures(wl, res, "van")[0]
    fails += (emu.bitwise_failures if gt <= 2 else emu.close_failures)(res, "dtd", "van")
    assert not fails, "\n".join(fails[:40])


@pytest.mark.parametrize("gt,gep", [(2, 2), (1, 4), (4, 1)])
def test_emulated_gating_variants(gt, gep):
    """Top-2 (R22) + random token selection (R20) + aux loss (R21) through the exchange."""
    wl = emu.Workload(_shape(gt, gep, cf=0.75))
    flags = MOE_F_RANDOM_PRIORITY | MOE_F_AUX_LOSS
    modes = {"dtd": wl.config(True, flags, aux_loss_coef=0.03, top_k=2),
             "van": wl.config(False, flags, aux_loss_coef=0.03, top_k=2)}
    res = emu.run_modes(wl, modes, seed=4242)
    fails = emu.oracle_failures(wl, res, "dtd", top2=True, seed=4242, aux_coef=0.03)[0]
    fails += (emu.bitwise_failures if gt <= 2 else emu.close_failures)(res, "dtd", "van")
    assert not fails, "\n".join(fails[:40])


def test_emulated_data_parallel_replicas():
    """G_data = 2 over EP pairs (world 4): two independent EP groups, no cross-talk."""
    wl = emu.Workload(_shape(1, 2), gd=2)
    res = emu.run_modes(wl, {"dtd": wl.config(True)})
    fails = emu.oracle_failures(wl, res, "dtd")[0]
    assert not fails, "\n".join(fails[:40])


# ---------------------------------------------------------------- ring / schedules
def _schedule_ffbb(order):
    """Forwards and backwards of several microbatches in `order` (e.g. F0 F1 B0 B1)."""

    def run(layer, inp, st):
        x, wg, w1, w2 = inp["x"], inp["wg"], inp["w1"], inp["w2"]
        outs, saved, errors = {}, {}, {}
        for op, mb in order:
            xm = x if mb % 2 == 0 else torch.flip(x, dims=[0])  # microbatch 1: other tokens order
            dym = inp["dy"] if mb % 2 == 0 else torch.flip(inp["dy"], dims=[0])
            if op == "F":
                y, sv = layer.moe_forward(xm, wg, w1, w2, stream=st)
                saved[mb] = (y, sv)
            else:
                try:
                    g = layer.moe_backward(dym, saved[mb][1], xm, wg, w1, w2, stream=st)
                    outs[mb] = tuple(t.clone() for t in (saved[mb][0], *g))
                except MoEError as e:
                    errors[mb] = e.name
        st.synchronize()
        return {"outs": outs, "errors": errors}

    return run


@pytest.mark.parametrize("gt,gep", [(1, 2), (2, 2)])
def test_emulated_microbatches_in_flight(gt, gep):
    """F0 F1 B1 B0 and F0 B0 F1 B1 give the same bits per microbatch (ring slots, epochs and
    single-buffered backward windows reused across steps); three steps in a row too."""
    wl = emu.Workload(_shape(gt, gep))
    cfg = wl.config(True)
    seqs = {"serial": [("F", 0), ("B", 0), ("F", 1), ("B", 1), ("F", 0), ("B", 0)],
            "ffbb": [("F", 0), ("F", 1), ("B", 1), ("B", 0)],
            "ffbb2": [("F", 0), ("F", 1), ("B", 0), ("B", 1)]}
    got = {}
    for name, order in seqs.items():
        res = emu.run_modes(wl, {name: cfg}, schedule=_schedule_ffbb(order))
        got[name] = [rr[name] for rr in res]
    for r in range(wl.world):
        for name in ("ffbb", "ffbb2"):
            assert not got[name][r]["errors"], got[name][r]["errors"]
            for mb in (0, 1):
                for a, b in zip(got["serial"][r]["outs"][mb], got[name][r]["outs"][mb]):
                    assert torch.equal(a, b), (r, name, mb)
    # microbatch 0 of the serial run is the oracle-checked layer
    res = emu.run_modes(wl, {"dtd": cfg})
    fails = emu.oracle_failures(wl, res, "dtd")[0]
    assert not fails, "\n".join(fails[:20])
    for r in range(wl.world):
        for a, b in zip(got["serial"][r]["outs"][0], [res[r]["dtd"][k] for k in ("y", "dx", "dwg", "dw1", "dw2")]):
            assert torch.equal(a, b)


@pytest.mark.parametrize("depth", [2, 3])
def test_emulated_ring_depth(depth):
    """ring_depth forwards in flight are accepted; one more evicts the oldest, whose
    backward then returns MOE_ERR_STATE cleanly (the others still match bitwise)."""
    wl = emu.Workload(_shape(1, 2))
    cfg = wl.config(True, ring_depth=depth)
    order = [("F", 0), ("F", 1), ("F", 2), ("B", 2), ("B", 1), ("B", 0)]

    def sched(layer, inp, st):
        x, wg, w1, w2 = inp["x"], inp["wg"], inp["w1"], inp["w2"]
        saved, errors, outs = {}, {}, {}
        for op, mb in order:
            if op == "F":
                saved[mb] = layer.moe_forward(x, wg, w1, w2, stream=st)
            else:
                try:
                    g = layer.moe_backward(inp["dy"], saved[mb][1], x, wg, w1, w2, stream=st)
                    outs[mb] = tuple(t.clone() for t in g)
                except MoEError as e:
                    errors[mb] = e.name
        st.synchronize()
        return {"errors": errors, "outs": outs}

    res = emu.run_modes(wl, {"k": cfg}, schedule=sched)
    for r, rr in enumerate(res):
        e = rr["k"]["errors"]
        if depth >= 3:
            assert e == {}, e
        else:
            assert e == {0: "MOE_ERR_STATE"}, e
        for mb in rr["k"]["outs"]:
            for a, b in zip(rr["k"]["outs"][mb], rr["k"]["outs"][2]):
                assert torch.equal(a, b)


def test_emulated_shared_comm_plan_bytes_match_allocation():
    """moe_comm_plan_bytes == the device memory a communicator takes (within 1 MiB), for
    a communicator shared by layers of different sizes (windows sized for the largest)."""
    wl = emu.Workload(_shape(2, 2))
    big = wl.config(True, ring_depth=3).replace(tokens=8192, hidden=1024, ffn=1024)
    small = big.replace(hidden=256, ffn=512)
    plan = [moe_comm_plan_bytes([big, small], wl.world, r) for r in range(wl.world)]
    assert plan[0] == moe_comm_plan_bytes([big], wl.world, 0) > moe_comm_plan_bytes([small], wl.world, 0)
    for attempt in range(2):  # the first pass warms up the runtime's own allocations
        grp = EmuGroup(wl.world)
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        comms = emu.run_ranks(wl.world, lambda r: MoEComm([big, small], wl.world, r, emu=grp))
        torch.cuda.synchronize()
        used = free0 - torch.cuda.mem_get_info()[0]
        layers = emu.run_ranks(wl.world, lambda r: [MoELayer(c, comm=comms[r]) for c in (big, small)])
        for ls in layers:
            for layer in ls:
                layer.close()
        emu.run_ranks(wl.world, lambda r: comms[r].close())
        grp.close()
    assert abs(used - sum(plan)) <= (1 << 20), (used, sum(plan))


def test_emulated_absent_rank_times_out():
    """A rank that never calls moe_forward: its peers' forward returns MOE_ERR_TIMEOUT after
    peer_timeout_ms instead of hanging, and the context is poisoned afterwards."""
    import threading
    wl = emu.Workload(_shape(1, 2))
    cfg = wl.config(True, peer_timeout_ms=1500)
    done = threading.Event()

    def sched(layer, inp, st):
        if layer.rank == 1:  # alive (windows mapped) but never calls; leaves after rank 0
            done.wait(60)
            return {"skipped": True}
        x, wg, w1, w2 = inp["x"], inp["wg"], inp["w1"], inp["w2"]
        names = []
        for _ in range(2):
            try:
                layer.moe_forward(x, wg, w1, w2, stream=st)
                names.append("MOE_OK")
            except MoEError as e:
                names.append(e.name)
        st.synchronize()
        done.set()
        return {"names": names}

    res = emu.run_modes(wl, {"k": cfg}, schedule=sched)
    assert res[0]["k"]["names"] == ["MOE_ERR_TIMEOUT", "MOE_ERR_STATE"], res[0]


# ---------------------------------------------------------------- BASELINE shapes, 8 emulated ranks
@pytest.mark.parametrize("name,T", [("2.7b-ep8", 2048), ("6.7b-tp2ep4", 2048),
                                    ("2.7b-ep8", 16384), ("6.7b-tp2ep4", 16384)])
def test_emulated_baseline_shapes_sampled(name, T):
    """BASELINE configs[2] (2.7B, E 32, EP over 8) and configs[3] (6.7B, E 16, G_t = 2 x
    G_ep = 4, DTD vs vanilla) with all 8 ranks emulated, at T = 2048 per group and at the
    full T = 16384 the bench times: routing of every token bit-exact, y / dx on one token
    per (expert, 256-row M-tile), dW1 / dW2 on one f per 256-wide tile of every local
    expert of every rank (tests/emu.py sampled_failures)."""
    shape = synth.CONFIGS[name]
    wl = emu.Workload(shape, tokens=T)
    modes = {"dtd": wl.config(True)}
    if shape.g_tensor > 1:
        modes["van"] = wl.config(False)
    res = emu.run_modes(wl, modes)
    fails, errs = emu.sampled_failures(wl, res, "dtd")
    if "van" in modes:
        fails += emu.bitwise_failures(res, "dtd", "van")
        a2a = [(rr["dtd"]["stats"]["wire_bytes"]["a2a"], rr["van"]["stats"]["wire_bytes"]["a2a"]) for rr in res]
        fails += [f"a2a {d} x 2 != {v}" for d, v in a2a if d * 2 != v]
    assert not fails, "\n".join(fails[:40])
    print(name, T, "max rel L2", {k: max(v for kk, v in errs.items() if kk[-1] == k) for k in ("y", "dx", "dw1", "dw2")})
