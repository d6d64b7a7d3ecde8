"""Emulated-rank harness: every rank of a (G_t, G_ep, G_data) layout in THIS process on
ONE GPU (include/moe.h `moe_emu_group`), one host thread and one CUDA stream per rank,
each driving the product path through the C ABI (moe_comm_create_emulated,
moe_create_on_comm, moe_forward, moe_backward, ...).

What runs is the multi-GPU product code: the fused peer dispatch / combine-backward
(F3+F4+F5, B1+B2+B3), the split copy-engine exchange with per-source readiness
(G_t = 1), the fused TP-reduction + return kernel (F8+F9+F10, B7+B8+B9), the expert
GEMMs on strided source blocks, and the host-side piece lists, ring slots and ledger.
Only the publication differs from one process per GPU: a window barrier is a host
barrier plus cudaStreamWaitEvent on every rank's event, and a readiness flag is an
event — no kernel waits on another kernel (B200_PROFILING.md: spin kernels of several
ranks on one GPU can hang it).

The results are compared with the CPU oracle over all S = world / G_t token groups
(oracle.moe_oracle.layer with S groups; every expert receives every
group's tokens through the all-to-all).
"""
from __future__ import annotations

import threading
import traceback

import numpy as np
import torch

from oracle import moe_oracle as O
from paper_2305_13525_b200 import EmuGroup, MoEComm, MoEConfig, MoELayer, synth
from tests.helpers import REL_L2_BAR, bf16_tensor, parity_failures, rel_l2, tensor_f64

TEST_TIMEOUT_MS = 20000  # peer deadline inside the tests: a stuck rank fails fast


def coords(rank: int, gt: int, gep: int):
    """Rank r = (d*G_ep + ep)*G_t + t (R17) -> (d, ep, t)."""
    return rank // (gt * gep), (rank // gt) % gep, rank % gt


def run_ranks(world: int, fn, timeout: float = 900.0):
    """fn(rank) on `world` threads; returns the results, re-raises the first failure."""
    res, err = [None] * world, [None] * world

    def wrap(r):
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - reported below with the rank
            err[r] = (e, traceback.format_exc())

    th = [threading.Thread(target=wrap, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    if any(t.is_alive() for t in th):
        raise TimeoutError("emulated ranks did not finish")
    for r, e in enumerate(err):
        if e is not None:
            raise RuntimeError(f"rank {r} failed:\n{e[1]}") from e[0]
    return res


class Workload:
    """Seeded inputs of every token group (host bits) and every rank's device shards."""

    def __init__(self, shape: synth.LayerShape, gd: int = 1, skew: float = 1.0, tokens: int | None = None):
        self.shape = shape
        self.gt, self.gep, self.gd = shape.g_tensor, shape.g_expert, gd
        self.world = self.gt * self.gep * gd
        self.T = shape.tokens if tokens is None else tokens
        self.S = self.gep * gd  # token groups, numbered d*G_ep + ep
        self.xs = [synth.make_x(shape, s, self.T) for s in range(self.S)]
        self.dys = [synth.make_dy(shape, s, self.T) for s in range(self.S)]
        self.wg = synth.make_wg(shape, skew)
        self.w1, self.w2 = synth.make_experts(shape)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.rank_inputs = []
        for r in range(self.world):
            d, ep, t = coords(r, self.gt, self.gep)
            s = d * self.gep + ep
            w1s, w2s = synth.shard_experts(self.w1, self.w2, shape, ep, t)
            self.rank_inputs.append({"x": bf16_tensor(self.xs[s]), "dy": bf16_tensor(self.dys[s]),
                                     "wg": torch.from_numpy(self.wg).to(self.dev),
                                     "w1": bf16_tensor(w1s), "w2": bf16_tensor(w2s), "group": s})
        torch.cuda.synchronize()

    def config(self, dtd=True, flags=0, **kw) -> MoEConfig:
        sh = self.shape
        base = MoEConfig(self.T, sh.hidden, sh.ffn, sh.experts, sh.cf, self.gt, self.gep, dtd,
                         1 | flags, peer_timeout_ms=TEST_TIMEOUT_MS)
        return base.replace(**kw) if kw else base

    def oracle_arrays(self):
        return ([O.decode_bf16(a) for a in self.xs], [O.decode_bf16(a) for a in self.dys],
                self.wg.astype(np.float64), O.decode_bf16(self.w1), O.decode_bf16(self.w2))


def fwd_bwd(layer: MoELayer, inp: dict, stream, replay: bool = False, seed=None) -> dict:
    """One forward + backward of one rank on its stream; outputs cloned, stream synced."""
    if seed is not None:
        layer.moe_set_priority_seed(seed)
    x, dy, wg, w1, w2 = inp["x"], inp["dy"], inp["wg"], inp["w1"], inp["w2"]
    y, saved = layer.moe_forward(x, wg, w1, w2, stream=stream)
    if replay:
        layer.moe_forward_replay(saved, x, wg, w1, w2, stream=stream)
    dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wg, w1, w2, stream=stream)
    rt = layer.moe_routing(saved, stream=stream)
    out = {"y": y.clone(), "dx": dx.clone(), "dwg": dwg.clone(), "dw1": dw1.clone(), "dw2": dw2.clone()}
    aux = layer.moe_aux_loss(saved, stream=stream) if layer.cfg.flags & 128 else None
    stream.synchronize()
    out["rt"] = {k: v.cpu().numpy() for k, v in rt.items()}
    out["aux"] = None if aux is None else float(aux.item())
    out["stats"] = layer.moe_stats()
    out["layout"] = layer.layout
    return out


def run_modes(wl: Workload, modes: dict, replay_keys=(), seed=None, schedule=None) -> list[dict]:
    """Every mode (key -> MoEConfig) as one layer context on ONE shared communicator per
    rank (moe_comm planned for all of them), forward+backward each. Returns per-rank
    {key: outputs}."""
    grp = EmuGroup(wl.world)
    cfgs = list(modes.values())

    def rank_fn(r):
        torch.cuda.set_device(wl.dev)
        st = torch.cuda.Stream(device=wl.dev)
        out = {}
        with torch.cuda.stream(st):
            comm = MoEComm(cfgs, wl.world, r, emu=grp)
            try:
                for key, cfg in modes.items():
                    layer = MoELayer(cfg, comm=comm, device=wl.dev)
                    try:
                        if schedule is not None:
                            out[key] = schedule(layer, wl.rank_inputs[r], st)
                        else:
                            out[key] = fwd_bwd(layer, wl.rank_inputs[r], st, key in replay_keys, seed)
                    finally:
                        layer.close()
            finally:
                comm.close()
        return out

    try:
        return run_ranks(wl.world, rank_fn)
    finally:
        grp.close()


def _f64(t):
    return tensor_f64(t) if t.dtype == torch.bfloat16 else t.detach().cpu().numpy().astype(np.float64)


def oracle_failures(wl: Workload, res: list[dict], key: str, top2: bool = False, seed=None,
                    aux_coef: float = 0.0, rows: bool = True) -> tuple[list[str], dict]:
    """Compares every rank's outputs of mode `key` with the oracle over its EP group's S
    token groups: routing (tie protocol), slots and counts bit-exact; y / dx / dWg of the
    group and dW1 / dW2 of the shard within rel L2 1e-2 globally and 5e-2 per row, exact
    zeros where the oracle is zero; the G_t ranks of a group hold bitwise-identical y/dx/dWg."""
    from oracle import top2_oracle as T2
    fails, errs = [], {}
    xs, dys, wg, w1, w2 = wl.oracle_arrays()
    cf = wl.shape.cf
    order = None if seed is None else O.priority_order(wl.T, seed)
    for d in range(wl.gd):
        groups = [d * wl.gep + ep for ep in range(wl.gep)]
        overrides = []
        for ep, s in enumerate(groups):
            g = res[(d * wl.gep + ep) * wl.gt][key]["rt"]  # rank (d, ep, t = 0)
            if top2:
                r0 = T2.route_top2(xs[s], wg, T2.capacity_top2(wl.T, wg.shape[1], cf, wl.gt), order=order)
                tie = (r0.gap < O.TIE_GAP) | (g["gap"] < O.TIE_GAP)
                bad = np.nonzero((g["expert"] != r0.experts).any(axis=1) & ~tie)[0]
            else:
                r0 = O.route(xs[s], wg, O.capacity(wl.T, wg.shape[1], cf, wl.gt), order=order)
                tie = (r0.gap < O.TIE_GAP) | (g["gap"] < O.TIE_GAP)
                bad = np.nonzero((g["expert"] != r0.expert) & ~tie)[0]
            if bad.size:
                fails.append(f"{key} group {s}: routing mismatch outside ties at {bad[:8]}")
            overrides.append((np.nonzero(tie)[0], g["expert"][tie]))
        sub = [xs[s] for s in groups], [dys[s] for s in groups]
        if top2:
            ref = T2.layer_top2(*sub, wg, w1, w2, cf, wl.gt, overrides=overrides, order=order, aux_coef=aux_coef)
        else:
            ref = O.layer(*sub, wg, w1, w2, cf, wl.gt, overrides=overrides, priority_seed=seed, aux_coef=aux_coef)
        for ep in range(wl.gep):
            for t in range(wl.gt):
                r = (d * wl.gep + ep) * wl.gt + t
                g = res[r][key]
                L = g["layout"]
                rr = ref["routing"][ep]
                if not np.array_equal(g["rt"]["slot"], rr.slot):
                    fails.append(f"{key} rank {r}: slot mismatch")
                if not np.array_equal(g["rt"]["count"], rr.count):
                    fails.append(f"{key} rank {r}: count mismatch")
                El, Fl = L["experts_local"], L["ffn_local"]
                es, fs = slice(ep * El, (ep + 1) * El), slice(t * Fl, (t + 1) * Fl)
                pairs = {"y": (g["y"], ref["y"][ep]), "dx": (g["dx"], ref["dx"][ep]),
                         "dwg": (g["dwg"], ref["dwg"][ep]), "dw1": (g["dw1"], ref["dw1"][es, fs, :]),
                         "dw2": (g["dw2"], ref["dw2"][es, :, fs])}
                for name, (got, want) in pairs.items():
                    gv = _f64(got)
                    errs[(r, name)] = rel_l2(gv, want)
                    fails += [f"{key} rank {r} {m}" for m in
                              parity_failures(name, gv, want, rows=rows and name != "dwg")]
                if aux_coef and abs(g["aux"] - ref["aux"][ep]) > 1e-5 * abs(ref["aux"][ep]):
                    fails.append(f"{key} rank {r}: aux {g['aux']} vs {ref['aux'][ep]}")
                if t > 0:  # replicated outputs of the TP group are identical
                    g0 = res[r - t][key]
                    for name in ("y", "dx", "dwg"):
                        if not torch.equal(g[name], g0[name]):
                            fails.append(f"{key} rank {r}: {name} differs from rank {r - t} (same TP group)")
    return fails, errs


def bitwise_failures(res: list[dict], a: str, b: str, names=("y", "dx", "dwg", "dw1", "dw2")) -> list[str]:
    out = []
    for r, rr in enumerate(res):
        for n in names:
            if not torch.equal(rr[a][n], rr[b][n]):
                out.append(f"rank {r}: {a} != {b} (bitwise) for {n}")
    return out


def close_failures(res: list[dict], a: str, b: str, bar: float = REL_L2_BAR) -> list[str]:
    out = []
    for r, rr in enumerate(res):
        for n in ("y", "dx", "dwg", "dw1", "dw2"):
            e = rel_l2(_f64(rr[a][n]), _f64(rr[b][n]))
            if not e <= bar:
                out.append(f"rank {r}: {a} vs {b} rel L2 {e:.3e} for {n}")
    return out


def sampled_failures(wl: Workload, res: list[dict], key: str, seed: int = 0) -> tuple[list[str], dict]:
    """Full-size parity (top-1) without the full oracle layer: routing of every token
    (tie protocol), slots and counts bit-exact on every rank; y / dx on stratified tokens
    (one per (expert, 256-row M-tile) of the GEMM rows, plus dropped ones); dW1 rows / dW2
    columns on one f per 256-wide tile of every local expert of every rank. Each bound:
    rel L2 <= 1e-2 over the samples and <= 5e-2 per sampled row, exact zeros where the
    oracle is zero. (dWg needs dp of every token and is checked at reduced sizes.)"""
    from tests.helpers import LazyExperts, stratified_f, stratified_tokens
    fails, errs = [], {}
    wg = wl.wg.astype(np.float64)
    E = wg.shape[1]
    cap = O.capacity(wl.T, E, wl.shape.cf, wl.gt)
    w1, w2 = LazyExperts(wl.w1), LazyExperts(wl.w2)
    for d in range(wl.gd):
        groups = [d * wl.gep + ep for ep in range(wl.gep)]
        xs = [O.decode_bf16(wl.xs[s]) for s in groups]
        dys = [O.decode_bf16(wl.dys[s]) for s in groups]
        routings = []
        for ep, s in enumerate(groups):
            g = res[(d * wl.gep + ep) * wl.gt][key]["rt"]
            r0 = O.route(xs[ep], wg, cap)
            tie = (r0.gap < O.TIE_GAP) | (g["gap"] < O.TIE_GAP)
            bad = np.nonzero((g["expert"] != r0.expert) & ~tie)[0]
            if bad.size:
                fails.append(f"{key} group {s}: routing mismatch outside ties at {bad[:8]}")
            routings.append(O.route(xs[ep], wg, cap, override=(np.nonzero(tie)[0], g["expert"][tie])))
        for ep, r in enumerate(routings):
            for t in range(wl.gt):
                g = res[(d * wl.gep + ep) * wl.gt + t][key]
                if not np.array_equal(g["rt"]["slot"], r.slot) or not np.array_equal(g["rt"]["count"], r.count):
                    fails.append(f"{key} rank {(d * wl.gep + ep) * wl.gt + t}: slots/counts differ")
            toks = stratified_tokens(r, ep, seed=seed)
            yr, dxr = O.tokens_forward_backward(toks, xs[ep], dys[ep], wg, w1, w2, r)
            g = res[(d * wl.gep + ep) * wl.gt][key]
            for name, got, want in (("y", g["y"], yr), ("dx", g["dx"], dxr)):
                gv = tensor_f64(got[torch.from_numpy(toks).to(got.device)])
                errs[(d, ep, name)] = rel_l2(gv, want)
                fails += [f"{key} group {groups[ep]} {m}" for m in parity_failures(name, gv, want)]
        for ep in range(wl.gep):
            for t in range(wl.gt):
                rank = (d * wl.gep + ep) * wl.gt + t
                g = res[rank][key]
                El, Fl = g["layout"]["experts_local"], g["layout"]["ffn_local"]
                fl = stratified_f(Fl, seed=seed + rank)
                got1, want1, got2, want2 = [], [], [], []
                d1, d2 = g["dw1"], g["dw2"]
                for el in range(El):
                    e = ep * El + el
                    for f in fl:
                        a, b = O.expert_row_grads(e, t * Fl + int(f), xs, dys, w1, w2, routings)
                        want1.append(a)
                        want2.append(b)
                    fi = torch.from_numpy(fl).to(d1.device)
                    got1.append(tensor_f64(d1[el].index_select(0, fi)))
                    got2.append(tensor_f64(d2[el].index_select(1, fi).t()))
                for name, got, want in (("dw1", np.concatenate(got1), np.array(want1)),
                                        ("dw2", np.concatenate(got2), np.array(want2))):
                    errs[(rank, name)] = rel_l2(got, want)
                    fails += [f"{key} rank {rank} {m}" for m in parity_failures(name, got, want)]
    return fails, errs
