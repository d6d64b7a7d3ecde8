"""C ABI (CPU, no GPU needed): the library loads, exports every symbol of
include/moe.h, validates configs, and its host-side plan/ledger obeys the
invariants the paper fixes for DTD and the
collective counts."""
import ctypes
import os
import re

import pytest

from paper_2305_13525_b200 import MoEConfig, MoEError, binding, synth
from paper_2305_13525_b200 import moe_plan_bytes, moe_plan_collectives, moe_plan_layout
from paper_2305_13525_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def header_symbols():
    inc = os.path.join(ROOT, "include")
    src = "".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc)) if f.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = binding.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(binding.EXPORTS)


def test_status_strings():
    L = binding.lib()
    names = [L.moe_status_string(i).decode() for i in range(9)]
    assert names == ["MOE_OK", "MOE_ERR_ARG", "MOE_ERR_SHAPE", "MOE_ERR_ALIGN", "MOE_ERR_STATE",
                     "MOE_ERR_CUDA", "MOE_ERR_NCCL", "MOE_ERR_UNSUPPORTED", "MOE_ERR_TIMEOUT"]


@pytest.mark.parametrize("kw,status", [
    (dict(hidden=100), "MOE_ERR_SHAPE"),                      # H % 64
    (dict(ffn=8192 + 64, g_tensor=2), "MOE_ERR_SHAPE"),       # (F/G_t) % 64
    (dict(experts=16, g_expert=3), "MOE_ERR_SHAPE"),          # E % G_ep
    (dict(experts=65), "MOE_ERR_SHAPE"),                      # E <= 64
    (dict(tokens=0), "MOE_ERR_ARG"),
    (dict(capacity_factor=0.0), "MOE_ERR_ARG"),
    (dict(flags=512), "MOE_ERR_ARG"),  # first unused flag bit
    (dict(flags=128, aux_loss_coef=-1.0), "MOE_ERR_ARG"),
    (dict(top_k=3), "MOE_ERR_ARG"),
    (dict(top_k=2, experts=1), "MOE_ERR_SHAPE"),
    (dict(top_k=2, flags=2), "MOE_ERR_UNSUPPORTED"),        # forced routing is top-1 only
])
def test_config_validation(kw, status):
    base = dict(tokens=16384, hidden=2048, ffn=8192, experts=16)
    base.update(kw)
    cfg = MoEConfig(**base)
    with pytest.raises(MoEError) as ei:
        moe_plan_bytes(cfg, 1, 0)
    assert ei.value.name == status and ei.value.detail


def test_top2_capacity_and_saved_bytes():
    """R22: C = ceil(cf * 2T / E) (rounded to G_t); per-token routing arrays double."""
    from oracle import top2_oracle as T2
    for T, E, cf, gt in [(16384, 16, 1.0, 1), (1000, 5, 0.7, 1), (4096, 16, 1.25, 2)]:
        c2 = MoEConfig(T, 2048, 8192, E, cf, gt, 1, top_k=2)
        assert moe_plan_layout(c2, gt, 0)["capacity"] == T2.capacity_top2(T, E, cf, gt)
    one = moe_plan_bytes(MoEConfig(16384, 2048, 8192, 16), 1, 0)[0]
    two = moe_plan_bytes(MoEConfig(16384, 2048, 8192, 16, top_k=2), 1, 0)[0]
    assert two > one  # twice the slot space plus the [T][2] routing arrays


def test_world_must_factor():
    cfg = MoEConfig(16384, 2048, 8192, 16, 1.0, 2, 4)
    with pytest.raises(MoEError) as ei:
        moe_plan_layout(cfg, 6, 0)
    assert ei.value.name == "MOE_ERR_SHAPE"
    with pytest.raises(MoEError):
        moe_plan_layout(cfg, 8, 8)


def test_layout_rank_grid_and_capacity():
    cfg = MoEConfig.from_shape(synth.CONFIGS["6.7b-tp2ep4"])
    seen = set()
    for r in range(8):
        L = moe_plan_layout(cfg, 8, r)
        # rank = (d*G_ep + ep)*G_t + t, TP fastest (R17)
        assert r == (L["d"] * 4 + L["ep"]) * 2 + L["t"]
        seen.add((L["ep"], L["t"]))
        assert L["experts_local"] == 4 and L["ffn_local"] == 8192
        assert L["capacity"] == 1024 and L["slot_slice"] == 512 and L["rows_per_expert"] == 4096
        assert L["token_groups"] == 4
    assert len(seen) == 8
    # capacity rounding to a multiple of G_tensor (reading R2)
    L = moe_plan_layout(MoEConfig(100, 64, 256, 3, 1.0, 4, 1), 4, 0)
    assert L["capacity"] == 36 and L["slot_slice"] == 9


def test_plan_bytes_scale():
    cfg = MoEConfig.from_shape(synth.CONFIGS["1.3b"])
    saved, scratch = moe_plan_bytes(cfg)
    X = 16 * 1024 * 2048 * 2
    ffn = 16 * 1024 * 8192 * 2
    assert saved >= 2 * X + 2 * ffn            # X, O, Hpre, A
    assert saved < 2 * X + 2 * ffn + (8 << 20)
    assert scratch >= X + ffn                  # dY + dHpre at least


def _sched(shape, dtd, world=None):
    cfg = MoEConfig.from_shape(shape, dtd=dtd)
    return moe_plan_collectives(cfg, world or shape.world, 0)


def _a2a_bytes(s):
    return sum(c["wire_bytes"] for c in s if c["kind"] == "a2a")


@pytest.mark.parametrize("gt,gep", [(2, 4), (4, 2), (2, 2), (4, 4), (8, 1), (2, 8)])
def test_dtd_cuts_a2a_bytes_by_g_tensor_exactly(gt, gep):
    shape = synth.LayerShape("s", 16384, 2560, 10240, 32, 1.0, gt, gep)
    van, dtd = _sched(shape, False), _sched(shape, True)
    assert _a2a_bytes(dtd) * gt == _a2a_bytes(van)        # PAPER.md:1125-1126 / SPEC.md:557


def test_collective_counts_per_layer():
    shape = synth.CONFIGS["6.7b-tp2ep4"]
    van, dtd = _sched(shape, False), _sched(shape, True)
    kinds = lambda s, p: [c["kind"] for c in s if c["pass"] == p]  # noqa: E731
    # vanilla: "two all-reduce calls ... and two all-to-all calls", repeated in backward
    # (PAPER.md:1094-1096): here the MoE layer's own share is 2 a2a + 1 AR per pass
    # (the attention all-reduce (2) of Fig. tp-ep-dp is outside the layer).
    assert kinds(van, "forward") == ["a2a", "allreduce", "a2a"]
    assert kinds(van, "backward") == ["a2a", "allreduce", "a2a"]
    # DTD: drop -> a2a -> all-gather; AR + drop = reduce-scatter; backward swaps
    assert kinds(dtd, "forward") == ["a2a", "allgather", "reducescatter", "a2a", "allgather"]
    assert kinds(dtd, "backward") == ["a2a", "allgather", "reducescatter", "a2a", "allgather"]
    # single GPU: no collectives at all
    assert _sched(synth.CONFIGS["1.3b"], True) == []


def test_allgather_bytes_formula_and_egress_accounting():
    shape = synth.CONFIGS["6.7b-tp2ep4"]
    dtd = _sched(shape, True)
    for c in dtd:
        if c["kind"] in ("allgather", "reducescatter"):
            s = c["group_size"]
            assert c["wire_bytes"] * s == c["buffer_bytes"] * (s - 1)
    # per-rank forward egress in units of X = E*C*H*2
    X = 16 * 1024 * 4096 * 2
    fwd = lambda s: sum(c["wire_bytes"] for c in s if c["pass"] == "forward")  # noqa: E731
    assert fwd(_sched(shape, False)) == int(2.5 * X)
    assert fwd(dtd) == int(2.25 * X)


def test_golden_dtd_example():
    """PAPER.md:1151-1152 (Fig. dtd): a TP pair holding {a1, a2}; GPU 0 keeps a1,
    GPU 1 keeps a2 — slot-range slices of C = 2 (reading R10); SPEC.md:539-542's
    all-gather arithmetic for 1 token of H elements at 2 bytes."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "dtd_pair.txt")) if l.strip() and not l.startswith("#")]
    kv = {r[0]: int(r[1]) for r in rows}
    H, gt = kv["hidden"], kv["g_tensor"]
    cfg = MoEConfig(kv["tokens"], 64, 128, kv["experts"], 1.0, gt, 1, True)
    lay = [moe_plan_layout(cfg, gt, r) for r in range(gt)]
    assert lay[0]["capacity"] == kv["capacity"] and lay[0]["slot_slice"] == kv["slot_slice"]
    # slot c of the expert is kept by TP rank c // C_s
    assert [c // lay[0]["slot_slice"] for c in range(kv["capacity"])] == [kv["keeper_a1"], kv["keeper_a2"]]
    full = kv["tokens"] * H * 2
    assert full * (gt - 1) // gt == kv["allgather_rx_bytes"]


@pytest.mark.parametrize("gt,gep,dtd", [(2, 4, False), (2, 4, True), (1, 8, True), (4, 2, True)])
def test_cac_cuts_collective_calls_by_one_third(gt, gep, dtd):
    """SPEC.md:559 / PAPER.md:1181-1188: with activation checkpointing the replay repeats
    the forward's collectives (fwd + replay + bwd); CAC replays from the stash with none,
    so calls and bytes drop by exactly 1/3 and the replay moves 0 bytes."""
    from paper_2305_13525_b200 import MOE_F_CAC, MOE_F_CHECKPOINT
    base = MoEConfig(16384, 2560, 10240, 32, 1.0, gt, gep, dtd)
    ck = MoEConfig(16384, 2560, 10240, 32, 1.0, gt, gep, dtd, base.flags | MOE_F_CHECKPOINT)
    cac = MoEConfig(16384, 2560, 10240, 32, 1.0, gt, gep, dtd, base.flags | MOE_F_CHECKPOINT | MOE_F_CAC)
    w = gt * gep
    s0, s1, s2 = (moe_plan_collectives(c, w, 0) for c in (base, ck, cac))
    assert s2 == s0                                   # CAC: exactly the un-checkpointed schedule
    replay = [c for c in s1 if c["pass"] == "replay"]
    assert [c["kind"] for c in replay] == [c["kind"] for c in s0 if c["pass"] == "forward"]
    assert len(s2) * 3 == len(s1) * 2
    tot = lambda s: sum(c["wire_bytes"] for c in s)  # noqa: E731
    assert tot(s2) * 3 == tot(s1) * 2
    assert [c["pass"] for c in s1][: len(replay) * 2] == ["forward"] * len(replay) + ["replay"] * len(replay)


def test_checkpoint_saved_blob_drops_activations():
    from paper_2305_13525_b200 import MOE_F_CAC, MOE_F_CHECKPOINT
    base = MoEConfig.from_shape(synth.CONFIGS["1.3b"])
    ck = MoEConfig(base.tokens, base.hidden, base.ffn, base.experts, 1.0, 1, 1, True,
                   base.flags | MOE_F_CHECKPOINT | MOE_F_CAC)
    s0, _ = moe_plan_bytes(base)
    s1, sc1 = moe_plan_bytes(ck)
    ffn = 16 * 1024 * 8192 * 2
    assert s0 - s1 == 2 * ffn           # G and A are re-materialized by the replay
    with pytest.raises(MoEError):       # CAC without checkpointing is rejected
        moe_plan_bytes(MoEConfig(base.tokens, base.hidden, base.ffn, base.experts, flags=1 | MOE_F_CAC))


# ---------------------------------------------------------------- shared communicator (host plan)
def _mib2(b):
    return (b + (2 << 20) - 1) // (2 << 20) * (2 << 20)


def test_comm_plan_bytes_window_formula():
    """Window memory of a communicator (include/moe.h moe_comm_plan_bytes): a ring of
    ring_depth (X, O) window pairs + dY, dS (+ the two TP-partial windows when G_t > 1) +
    the flag page and metadata, each rounded to the 2 MiB allocation granularity."""
    from paper_2305_13525_b200 import moe_comm_plan_bytes
    cfg = MoEConfig.from_shape(synth.CONFIGS["6.7b-tp2ep4"])
    L = moe_plan_layout(cfg, 8, 0)
    xe = L["experts_local"] * L["rows_per_expert"] * 4096 * 2      # expert space [E_l][R][H]
    so = 16 * L["capacity"] * 4096 * 2                               # slot space [E][C][H]
    d2 = moe_comm_plan_bytes([cfg], 8, 0)
    d3 = moe_comm_plan_bytes([cfg.replace(ring_depth=3)], 8, 0)
    assert d3 - d2 == _mib2(xe) + _mib2(so)                          # one more ring slot
    fixed = d2 - 3 * _mib2(xe) - 3 * _mib2(so) - 2 * _mib2(xe)      # X,O ring + dY, dS + Y, dXp
    assert 0 < fixed <= 2 * (2 << 20)                                # flags + metadata
    # G_t = 1: no TP-partial windows
    ep = MoEConfig.from_shape(synth.CONFIGS["2.7b-ep8"])
    L = moe_plan_layout(ep, 8, 0)
    xe = L["experts_local"] * L["rows_per_expert"] * 2560 * 2
    so = 32 * L["capacity"] * 2560 * 2
    assert moe_comm_plan_bytes([ep], 8, 0) - 3 * _mib2(xe) - 3 * _mib2(so) <= 2 * (2 << 20)


def test_comm_plan_shared_by_layers_does_not_scale_with_layer_count():
    from paper_2305_13525_b200 import moe_comm_plan_bytes
    cfg = MoEConfig.from_shape(synth.CONFIGS["6.7b-tp2ep4"])
    one = moe_comm_plan_bytes([cfg], 8, 3)
    assert moe_comm_plan_bytes([cfg] * 24, 8, 3) == one
    small = cfg.replace(hidden=1024, ffn=4096)
    assert moe_comm_plan_bytes([cfg, small], 8, 3) == one            # sized for the largest
    assert moe_comm_plan_bytes([small], 8, 3) < one


def test_comm_plan_no_windows_without_peer_exchange():
    from paper_2305_13525_b200 import MOE_F_NCCL_EXCHANGE, moe_comm_plan_bytes
    cfg = MoEConfig.from_shape(synth.CONFIGS["6.7b-tp2ep4"])
    assert moe_comm_plan_bytes([cfg.replace(flags=cfg.flags | MOE_F_NCCL_EXCHANGE)], 8, 0) == 0
    assert moe_comm_plan_bytes([MoEConfig.from_shape(synth.CONFIGS["1.3b"])], 1, 0) == 0


@pytest.mark.parametrize("kw,status", [
    (dict(ring_depth=-1), "MOE_ERR_ARG"),
    (dict(ring_depth=65), "MOE_ERR_ARG"),
    (dict(peer_timeout_ms=-5), "MOE_ERR_ARG"),
])
def test_comm_config_validation(kw, status):
    cfg = MoEConfig(4096, 256, 512, 8, 1.0, 2, 2, True, **kw)
    with pytest.raises(MoEError) as ei:
        moe_plan_layout(cfg, 4, 0)
    assert ei.value.name == status


def test_comm_plan_rejects_mixed_layouts():
    from paper_2305_13525_b200 import moe_comm_plan_bytes
    a = MoEConfig(4096, 256, 512, 8, 1.0, 2, 2, True)
    with pytest.raises(MoEError) as ei:
        moe_comm_plan_bytes([a, a.replace(g_tensor=1, g_expert=4)], 4, 0)
    assert ei.value.name == "MOE_ERR_ARG"


def test_peer_dtd_beyond_eight_tp_ranks_is_unsupported():
    """The fused peer dispatch resolves at most 8 destination rows per slot (G_t <= 8);
    larger DTD groups must use the NCCL exchange instead of silently dropping rows."""
    from paper_2305_13525_b200 import MOE_F_NCCL_EXCHANGE
    cfg = MoEConfig(4096, 256, 16 * 64, 16, 1.0, 16, 1, True)
    with pytest.raises(MoEError) as ei:
        moe_plan_layout(cfg, 16, 0)
    assert ei.value.name == "MOE_ERR_UNSUPPORTED"
    moe_plan_layout(cfg.replace(flags=cfg.flags | MOE_F_NCCL_EXCHANGE), 16, 0)
    moe_plan_layout(cfg.replace(dtd=False), 16, 0)


def test_nvls_plan_allgather_egress():
    """MOE_F_NVLS (PAPER.md:1153-1158 with the all-gather on NVLink SHARP multicast): the same
    collective calls and a2a bytes as folded DTD; each all-gather's wire bytes are the rank's
    own slice once instead of G_t - 1 copies."""
    from paper_2305_13525_b200 import MOE_F_NVLS
    for gt, gep in ((2, 2), (4, 1), (4, 2)):
        base = MoEConfig(tokens=4096, hidden=512, ffn=1024, experts=8, g_tensor=gt, g_expert=gep)
        nv = MoEConfig(tokens=4096, hidden=512, ffn=1024, experts=8, g_tensor=gt, g_expert=gep,
                       flags=base.flags | MOE_F_NVLS)
        world = gt * gep
        for rank in range(world):
            a, b = moe_plan_collectives(base, world, rank), moe_plan_collectives(nv, world, rank)
            assert [(c["kind"], c["pass"], c["step"]) for c in a] == [(c["kind"], c["pass"], c["step"]) for c in b]
            for ca, cb in zip(a, b):
                if ca["kind"] == "allgather":
                    assert cb["wire_bytes"] * (gt - 1) == ca["wire_bytes"]
                else:
                    assert cb["wire_bytes"] == ca["wire_bytes"]
