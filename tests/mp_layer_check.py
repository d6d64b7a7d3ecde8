"""Multi-rank MoE-layer parity (launched by tests/test_gpu_multi.py under torchrun).

Every rank builds its shard of a seeded workload (all token groups are generated
on the host), runs moe_forward/moe_backward through the C ABI with DTD and
without, and checks against the CPU oracle computed locally for all groups:
  * routing bit-exact outside logged ties; slots/counts bit-exact after the
    tie-override protocol;
  * y, dx, dWg of its token group and dW1/dW2 of its expert shard within
    relative L2 1e-2 (BASELINE.json);
  * DTD output == vanilla output bitwise for G_tensor <= 2;
  * a2a wire bytes: vanilla == G_tensor x DTD, exactly.
Exit code 0 iff every rank passed.

    torchrun --nproc-per-node N tests/mp_layer_check.py --gt 2 --gep 2 --tokens 512
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import moe_oracle as O  # noqa: E402
from paper_2305_13525_b200 import (MOE_F_AUX_LOSS, MOE_F_CAC, MOE_F_CHECKPOINT,  # noqa: E402
                                   MOE_F_NCCL_EXCHANGE, MOE_F_NVLS, MOE_F_RANDOM_PRIORITY, MoEConfig, MoEError,
                                   MoELayer, synth)
from tests.helpers import REL_L2_BAR, bf16_tensor, rel_l2, tensor_f64  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gt", type=int, default=1)
    ap.add_argument("--gep", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--ffn", type=int, default=512)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--cf", type=float, default=1.0)
    ap.add_argument("--variants", action="store_true",
                    help="also run top-2 + random priority + aux loss (NEXT #4), DTD and vanilla")
    a = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    shape = synth.LayerShape("mp", a.tokens, a.hidden, a.ffn, a.experts, a.cf, a.gt, a.gep)
    assert world % (a.gt * a.gep) == 0
    gd = world // (a.gt * a.gep)
    S = world // a.gt  # token groups
    failures = []

    # host inputs for every token group (groups numbered d*G_ep + ep)
    xs_b = [synth.make_x(shape, s) for s in range(S)]
    dys_b = [synth.make_dy(shape, s) for s in range(S)]
    wg = synth.make_wg(shape)
    w1_b, w2_b = synth.make_experts(shape)

    results = {}
    # (dtd, extra flags, key): DTD, vanilla, NCCL-exchange baseline, checkpointing with and without CAC
    modes = ((True, 0, True), (False, 0, False), (True, MOE_F_NCCL_EXCHANGE, "nccl"),
             (True, MOE_F_CHECKPOINT | MOE_F_CAC, "cac"), (True, MOE_F_CHECKPOINT, "ckpt"))
    if a.gt > 1:  # DTD's all-gathers on NVLink SHARP multicast (NEXT #2)
        modes += ((True, MOE_F_NVLS, "nvls"),)
    for dtd, extra, key in modes:
        cfg = MoEConfig.from_shape(shape, dtd=dtd)
        cfg = MoEConfig(cfg.tokens, cfg.hidden, cfg.ffn, cfg.experts, cfg.capacity_factor,
                        cfg.g_tensor, cfg.g_expert, cfg.dtd, cfg.flags | extra)
        try:
            layer = MoELayer(cfg, world, rank, dev)
        except MoEError as e:
            if key == "nvls" and "UNSUPPORTED" in str(e):
                print(f"[rank {rank}] NVLS unavailable: {e}", flush=True)
                continue
            raise
        L = layer.layout
        s = L["d"] * a.gep + L["ep"]
        w1s, w2s = synth.shard_experts(w1_b, w2_b, shape, L["ep"], L["t"])
        x = bf16_tensor(xs_b[s])
        dy = bf16_tensor(dys_b[s])
        wgt = torch.from_numpy(wg).to(dev)
        w1 = bf16_tensor(w1s)
        w2 = bf16_tensor(w2s)
        y, saved = layer.moe_forward(x, wgt, w1, w2)
        if extra & MOE_F_CHECKPOINT:
            layer.moe_forward_replay(saved, x, wgt, w1, w2)
        dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wgt, w1, w2)
        rt = layer.moe_routing(saved)
        torch.cuda.synchronize()
        st = layer.moe_stats()
        results[key] = {"y": y.clone(), "dx": dx.clone(), "dwg": dwg.clone(), "dw1": dw1.clone(),
                        "dw2": dw2.clone(), "rt": {k: v.cpu().numpy() for k, v in rt.items()},
                        "stats": st, "layout": L, "group": s}
        layer.close()

    L = results[True]["layout"]
    s = results[True]["group"]
    # ---- oracle over the EP group of this rank (G_data replicas are independent)
    d = L["d"]
    groups = [d * a.gep + ep for ep in range(a.gep)]
    xs = [O.decode_bf16(xs_b[g]) for g in groups]
    dys = [O.decode_bf16(dys_b[g]) for g in groups]
    w1d, w2d = O.decode_bf16(w1_b), O.decode_bf16(w2_b)
    wgd = wg.astype(np.float64)
    cap = O.capacity(a.tokens, a.experts, a.cf, a.gt)
    # tie protocol needs every group's GPU routing: gather expert/gap from the t == 0 ranks
    ge = torch.from_numpy(results[True]["rt"]["expert"]).to(dev)
    gg = torch.from_numpy(results[True]["rt"]["gap"]).to(dev)
    all_e = [torch.empty_like(ge) for _ in range(world)]
    all_g = [torch.empty_like(gg) for _ in range(world)]
    dist.all_gather(all_e, ge)
    dist.all_gather(all_g, gg)
    overrides = []
    for gi, g in enumerate(groups):
        r_rank = g * a.gt  # rank (d, ep, t=0) of group g
        ex = all_e[r_rank].cpu().numpy()
        gp = all_g[r_rank].cpu().numpy()
        r0 = O.route(xs[gi], wgd, cap)
        tie = (r0.gap < O.TIE_GAP) | (gp < O.TIE_GAP)
        bad = np.nonzero((ex != r0.expert) & ~tie)[0]
        if bad.size:
            failures.append(f"group {g}: routing mismatch outside ties at {bad[:8]}")
        overrides.append((np.nonzero(tie)[0], ex[tie]))
    ref = O.layer(xs, dys, wgd, w1d, w2d, a.cf, a.gt, overrides=overrides)
    gi = groups.index(s)
    r = ref["routing"][gi]
    g = results[True]
    if not (g["rt"]["slot"] == r.slot).all():
        failures.append("slot mismatch")
    if not (g["rt"]["count"] == r.count).all():
        failures.append("count mismatch")
    El, Fl = L["experts_local"], L["ffn_local"]
    es = slice(L["ep"] * El, (L["ep"] + 1) * El)
    fs = slice(L["t"] * Fl, (L["t"] + 1) * Fl)
    errs = {"y": rel_l2(tensor_f64(g["y"]), ref["y"][gi]),
            "dx": rel_l2(tensor_f64(g["dx"]), ref["dx"][gi]),
            "dwg": rel_l2(g["dwg"].cpu().numpy(), ref["dwg"][gi]),
            "dw1": rel_l2(tensor_f64(g["dw1"]), ref["dw1"][es, fs, :]),
            "dw2": rel_l2(tensor_f64(g["dw2"]), ref["dw2"][es, :, fs])}
    for k, v in errs.items():
        if not v <= REL_L2_BAR:
            failures.append(f"{k} rel L2 {v:.3e}")
    # ---- DTD vs vanilla
    v, t_ = results[False], results[True]
    for k in ("y", "dx", "dwg", "dw1", "dw2"):
        same = torch.equal(v[k], t_[k])
        if a.gt <= 2 and not same:
            failures.append(f"DTD != vanilla (bitwise) for {k}")
        if not same and rel_l2(tensor_f64(v[k]), tensor_f64(t_[k])) > 1e-2:
            failures.append(f"DTD vs vanilla differ for {k}")
    # ---- peer-memory exchange vs NCCL exchange (same arithmetic, same positions; the TP
    # sum of G_t > 2 partials is fixed-order fp32 in the peer kernel and NCCL's ring order in
    # NCCL mode, so bitwise only for G_t <= 2, where a + b is order-free)
    nc = results["nccl"]
    for k in ("y", "dx", "dwg", "dw1", "dw2"):
        if a.gt <= 2 and not torch.equal(nc[k], t_[k]):
            failures.append(f"peer exchange != NCCL exchange (bitwise) for {k}")
        if rel_l2(tensor_f64(nc[k]), tensor_f64(t_[k])) > 1e-2:
            failures.append(f"peer exchange vs NCCL exchange differ for {k}")
    if nc["stats"]["wire_bytes"] != t_["stats"]["wire_bytes"]:
        failures.append(f"ledger differs: peer {t_['stats']['wire_bytes']} nccl {nc['stats']['wire_bytes']}")
    # ---- checkpointing: replay (with / without CAC) reproduces the run bitwise; CAC's replay
    # issues no collective, plain checkpointing re-issues the forward's
    for key in ("cac", "ckpt"):
        for k in ("y", "dx", "dwg", "dw1", "dw2"):
            if not torch.equal(results[key][k], t_[k]):
                failures.append(f"{key} replay != un-checkpointed run (bitwise) for {k}")
    if results["cac"]["stats"]["replay_calls"] != 0:
        failures.append(f"CAC replay issued {results['cac']['stats']['replay_calls']} collectives")
    if results["ckpt"]["stats"]["replay_calls"] != t_["stats"]["forward_calls"]:
        failures.append("plain checkpoint replay did not repeat the forward's collectives")
    # ---- NVLS all-gathers: the same bits at the same positions as the folded DTD exchange,
    # a2a bytes unchanged, all-gather egress 1 / (G_t - 1) of the folded one
    if "nvls" in results:
        nv = results["nvls"]
        for k in ("y", "dx", "dwg", "dw1", "dw2"):
            if not torch.equal(nv[k], t_[k]):
                failures.append(f"NVLS != folded DTD (bitwise) for {k}")
        if nv["stats"]["wire_bytes"]["a2a"] != t_["stats"]["wire_bytes"]["a2a"]:
            failures.append("NVLS a2a bytes differ from DTD")
        ag_f, ag_n = t_["stats"]["wire_bytes"]["allgather"], nv["stats"]["wire_bytes"]["allgather"]
        if ag_n * (a.gt - 1) != ag_f:
            failures.append(f"NVLS all-gather egress {ag_n} x {a.gt - 1} != folded {ag_f}")
    a2a_dtd = t_["stats"]["wire_bytes"]["a2a"]
    a2a_van = v["stats"]["wire_bytes"]["a2a"]
    if a2a_dtd * a.gt != a2a_van:
        failures.append(f"a2a bytes: dtd {a2a_dtd} x {a.gt} != vanilla {a2a_van}")
    if a.variants:
        failures += check_variants(a, world, rank, dev, shape, xs_b, dys_b, wg, w1_b, w2_b)
    print(f"[rank {rank}] (d,ep,t)=({L['d']},{L['ep']},{L['t']}) errs="
          + " ".join(f"{k}={e:.2e}" for k, e in errs.items())
          + f" a2a dtd={a2a_dtd} van={a2a_van} calls={t_['stats']['calls']}"
          + (" FAIL: " + "; ".join(failures) if failures else " ok"), flush=True)
    flag = torch.tensor([len(failures)], device=dev)
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


def check_variants(a, world, rank, dev, shape, xs_b, dys_b, wg, w1_b, w2_b):
    """Top-2 (R22) with random priority (R20) and the aux loss (R21) through the exchange:
    parity with oracle/top2_oracle.py and DTD == vanilla bitwise (G_t <= 2)."""
    from oracle import top2_oracle as T2
    failures = []
    seed, coef = 4242, 0.03
    res = {}
    for dtd in (True, False):
        cfg = MoEConfig.from_shape(shape, dtd=dtd)
        cfg = MoEConfig(cfg.tokens, cfg.hidden, cfg.ffn, cfg.experts, cfg.capacity_factor, cfg.g_tensor,
                        cfg.g_expert, cfg.dtd, cfg.flags | MOE_F_RANDOM_PRIORITY | MOE_F_AUX_LOSS, coef, top_k=2)
        layer = MoELayer(cfg, world, rank, dev)
        layer.moe_set_priority_seed(seed)
        L = layer.layout
        s = L["d"] * a.gep + L["ep"]
        w1s, w2s = synth.shard_experts(w1_b, w2_b, shape, L["ep"], L["t"])
        x, dy = bf16_tensor(xs_b[s]), bf16_tensor(dys_b[s])
        wgt = torch.from_numpy(wg).to(dev)
        w1t, w2t = bf16_tensor(w1s), bf16_tensor(w2s)
        y, saved = layer.moe_forward(x, wgt, w1t, w2t)
        dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wgt, w1t, w2t)
        rt = layer.moe_routing(saved)
        aux = layer.moe_aux_loss(saved)
        torch.cuda.synchronize()
        res[dtd] = {"y": y, "dx": dx, "dwg": dwg, "dw1": dw1, "dw2": dw2, "aux": aux.item(),
                    "rt": {k: v.cpu().numpy() for k, v in rt.items()}, "L": L, "s": s}
        layer.close()
    g = res[True]
    L = g["L"]
    groups = [L["d"] * a.gep + ep for ep in range(a.gep)]
    xs = [O.decode_bf16(xs_b[q]) for q in groups]
    dys = [O.decode_bf16(dys_b[q]) for q in groups]
    ge = torch.from_numpy(g["rt"]["expert"]).to(dev)
    gg = torch.from_numpy(g["rt"]["gap"]).to(dev)
    all_e = [torch.empty_like(ge) for _ in range(world)]
    all_g = [torch.empty_like(gg) for _ in range(world)]
    dist.all_gather(all_e, ge)
    dist.all_gather(all_g, gg)
    cap = T2.capacity_top2(a.tokens, a.experts, a.cf, a.gt)
    order = O.priority_order(a.tokens, seed)
    overrides = []
    for gi, q in enumerate(groups):
        ex = all_e[q * a.gt].cpu().numpy()
        gp = all_g[q * a.gt].cpu().numpy()
        r0 = T2.route_top2(xs[gi], wg.astype(np.float64), cap, order=order)
        tie = (r0.gap < O.TIE_GAP) | (gp < O.TIE_GAP)
        if ((ex != r0.experts).any(axis=1) & ~tie).any():
            failures.append(f"variants: top-2 routing mismatch outside ties (group {q})")
        overrides.append((np.nonzero(tie)[0], ex[tie]))
    ref = T2.layer_top2(xs, dys, wg.astype(np.float64), O.decode_bf16(w1_b), O.decode_bf16(w2_b), a.cf, a.gt,
                        overrides=overrides, order=order, aux_coef=coef)
    gi = groups.index(g["s"])
    r = ref["routing"][gi]
    if not (g["rt"]["slot"] == r.slot).all():
        failures.append("variants: slot mismatch")
    El, Fl = L["experts_local"], L["ffn_local"]
    es = slice(L["ep"] * El, (L["ep"] + 1) * El)
    fs = slice(L["t"] * Fl, (L["t"] + 1) * Fl)
    errs = {"y": rel_l2(tensor_f64(g["y"]), ref["y"][gi]), "dx": rel_l2(tensor_f64(g["dx"]), ref["dx"][gi]),
            "dwg": rel_l2(g["dwg"].cpu().numpy(), ref["dwg"][gi]),
            "dw1": rel_l2(tensor_f64(g["dw1"]), ref["dw1"][es, fs, :]),
            "dw2": rel_l2(tensor_f64(g["dw2"]), ref["dw2"][es, :, fs])}
    for k, v in errs.items():
        if not v <= REL_L2_BAR:
            failures.append(f"variants: {k} rel L2 {v:.3e}")
    if abs(g["aux"] - ref["aux"][gi]) > 1e-5 * abs(ref["aux"][gi]):
        failures.append(f"variants: aux {g['aux']} vs {ref['aux'][gi]}")
    for k in ("y", "dx", "dwg", "dw1", "dw2"):
        if a.gt <= 2 and not torch.equal(res[True][k], res[False][k]):
            failures.append(f"variants: DTD != vanilla (bitwise) for {k}")
    print(f"[rank {rank}] variants errs=" + " ".join(f"{k}={e:.2e}" for k, e in errs.items()), flush=True)
    return failures


if __name__ == "__main__":
    main()
