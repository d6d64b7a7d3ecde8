#!/usr/bin/env python
"""MoE-layer fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1.3b|2.7b|6.7b] [--vanilla]

A step = one moe_forward + moe_backward through the C ABI (every §8(a) row)
over one batch of synthetic tokens. N = 1 runs BASELINE configs[1] (1.3B-shaped
layer, 16k tokens/GPU). N > 1 (torchrun, one process per GPU, NCCL) runs the
same per-GPU workload expert-parallel over N GPUs (E = 16 experts sharded,
16k tokens per GPU: weak scaling) unless --config picks the 2.7B / 6.7B
configs. Timing: W warm-up steps, then K steps between barrier +
synchronize, CUDA events on the launching stream, max over ranks. The working
set (>1 GB of expert weights per step) exceeds the 126 MB L2, so no flush.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_SEED = 230513525
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, choices=[None, "1.3b", "2.7b", "6.7b"])
    p.add_argument("--vanilla", action="store_true", help="disable DTD (G_tensor > 1 configs)")
    p.add_argument("--gt", type=int, default=None, help="G_tensor override (BASELINE scaling sweep)")
    p.add_argument("--nvls", action="store_true", help="DTD all-gathers on NVLink SHARP multicast (MOE_F_NVLS)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-optim", action="store_true", help="skip the tiled-optimizer measurement")
    return p.parse_args()


def measure_optimizer(dw1, dw2, peaks, steps, dev):
    """NEXT #3 (include/moe_optim.h): AdamW over this rank's expert parameters, whose bf16
    gradients the layer just produced (dW1, dW2). Fused (no temporary) vs the paper's
    tiled step (ts = 1.8 M, 4*ts-byte buffer, 2 launches per tile). Not part of `value`."""
    from paper_2305_13525_b200 import MOE_TILE_PARAMS_PAPER, moe_adamw_plan, moe_adamw_step
    n = dw1.numel() + dw2.numel()
    g = torch.cat([dw1.reshape(-1), dw2.reshape(-1)])
    gen = torch.Generator(device=dev).manual_seed(BASE_SEED + 7000)
    p = torch.randn(n, generator=gen, device=dev) * 0.02
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    p16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
    ts = MOE_TILE_PARAMS_PAPER
    n_tiles, temp_bytes = moe_adamw_plan(n, ts)
    temp = torch.empty(temp_bytes // 4, device=dev)
    hp = dict(lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    out = {"params": n, "tile_params": ts, "tiles": n_tiles, "temp_bytes_tiled": temp_bytes,
           "temp_bytes_untiled_upcast": 4 * n, "temp_bytes_fused": 0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(3, min(steps, 10))
    for name, tp, tmp, bpp, launches in (("fused", 0, None, 28, 1), ("tiled", ts, temp, 36, 2 * n_tiles)):
        for i in range(2):
            moe_adamw_step(g, p, m, v, p16, step=1 + i, tile_params=tp, temp=tmp, **hp)
        torch.cuda.synchronize()
        e0.record()
        for i in range(k):
            moe_adamw_step(g, p, m, v, p16, step=3 + i, tile_params=tp, temp=tmp, **hp)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        gbs = bpp * n / (ms / 1e3) / 1e9
        out[name] = {"ms": ms, "params_per_s": n / (ms / 1e3), "bytes_per_param": bpp, "GB/s": gbs,
                     "frac": gbs / peaks["hbm_gbs"], "launches": launches}
    return out


def workload(args, world):
    """(name, tokens/group, H, F, E, G_t, G_ep)."""
    cfg = args.config or "1.3b"
    shapes = {"1.3b": (2048, 8192, 16), "2.7b": (2560, 10240, 32), "6.7b": (4096, 16384, 16)}
    H, F, E = shapes[cfg]
    if args.gt:
        gt = args.gt
    elif cfg == "6.7b":
        gt = 2 if world >= 2 else 1
    else:
        gt = 1
    if world % gt:
        raise SystemExit(f"--gt {gt} does not divide {world} GPUs")
    gep = world // gt
    if cfg == "1.3b" and world == 1:
        name = "1.3b"
    elif gt == 1:
        name = f"{cfg}-ep{gep}"
    else:
        name = f"{cfg}-tp{gt}ep{gep}"
    return (name, 16384, H, F, E, gt, gep)


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x100: "display_clock", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                mask = int(parts[3], 16)
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if mask & bit:
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


class NvlinkCounter:
    """NVLink data bytes sent / received by this rank's GPU (NVML field counters, summed
    over links) around the timed region: the link-level evidence for the exchange bytes
    the library's ledger claims. None where NVML exposes no counter."""
    FIELDS = (("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", 1024,
               "NVML throughput data counters (KiB)"),
              ("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", 1,
               "NVML link byte counters"))

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.links = []
            for link in range(18):
                try:
                    if pynvml.nvmlDeviceGetNvLinkState(self.h, link) == pynvml.NVML_FEATURE_ENABLED:
                        self.links.append(link)
                except Exception:
                    pass
            for tx, rx, unit, what in self.FIELDS:
                ids = [(getattr(pynvml, tx), l) for l in self.links] + [(getattr(pynvml, rx), l) for l in self.links]
                vals = pynvml.nvmlDeviceGetFieldValues(self.h, ids)
                if self.links and all(v.nvmlReturn == 0 for v in vals):
                    self.ids, self.unit, self.what, self.ok = ids, unit, what, True
                    break
        except Exception:
            self.ok = False

    def read(self):
        if not self.ok:
            return None
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, self.ids)
        n = len(self.links)
        tx = sum(int(v.value.ullVal) for v in vals[:n]) * self.unit
        rx = sum(int(v.value.ullVal) for v in vals[n:]) * self.unit
        return tx, rx

    def delta(self, a, b, steps):
        if a is None or b is None:
            return {"unavailable": "NVML returns NOT_SUPPORTED for every NVLink byte counter on this "
                                   "system (tools/nvlink_probe.py); exchange bytes are the ledger's"}
        return {"tx_bytes_per_step": (b[0] - a[0]) / steps, "rx_bytes_per_step": (b[1] - a[1]) / steps,
                "links": len(self.links), "source": self.what}


def cpu_oracle_step(shape_t, sample_tokens, state):
    """One oracle fwd+bwd on a bounded token sample (same shapes; C scaled with T)."""
    from oracle import moe_oracle as O
    xs, dys, wg, w1, w2 = state
    t0 = time.perf_counter()
    O.layer(xs, dys, wg, w1, w2, 1.0, 1)
    return time.perf_counter() - t0


def oracle_state(H, F, E, tokens):
    from oracle import moe_oracle as O
    from paper_2305_13525_b200 import synth
    shape = synth.LayerShape("bench", tokens, H, F, E)
    x = O.decode_bf16(synth.make_x(shape, 0, tokens))
    dy = O.decode_bf16(synth.make_dy(shape, 0, tokens))
    wg = synth.make_wg(shape).astype(np.float64)
    w1, w2 = synth.make_experts(shape)
    return ([x], [dy], wg, O.decode_bf16(w1), O.decode_bf16(w2))


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def run_cpu_baseline(H, F, E, sample_tokens=256, budget_s=20.0):
    state = oracle_state(H, F, E, sample_tokens)
    cpu_oracle_step(None, sample_tokens, state)  # warm
    times = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(times) < 50:
        times.append(cpu_oracle_step(None, sample_tokens, state))
    dt = float(np.mean(times))
    return {"value": sample_tokens / dt, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"oracle fwd+bwd on {sample_tokens} tokens (H={H}, F={F}, E={E}, cf=1.0), "
                      f"mean of {len(times)} runs, float64 numpy"}


def reference_arm(args, world, rank):
    """The oracle, as it stands, on this host's cores (the only reference this
    tier has: /root/reference holds a paper, not code). Each step is a bounded
    token sample of the same workload, sized so W + K steps take ~2 minutes."""
    if rank != 0:
        return
    name, T, H, F, E, gt, gep = workload(args, world)  # the arm's config name; per-token math is the same
    probe = 64
    state = oracle_state(H, F, E, probe)
    t64 = cpu_oracle_step(None, probe, state)
    t64 = min(t64, cpu_oracle_step(None, probe, state))
    n = max(args.steps + args.warmup, 1)
    sample = int(max(16, min(256, probe * 120.0 / (n * max(t64, 1e-3)))))
    sample -= sample % 16
    if sample != probe:
        state = oracle_state(H, F, E, sample)
    for _ in range(args.warmup):
        cpu_oracle_step(None, sample, state)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_oracle_step(None, sample, state)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    v = sample / dt
    out = {"metric": "MoE-layer fwd+bwd tokens/s", "value": v, "unit": "tokens/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": name, "tokens_sample": sample, "hidden": H,
                                           "ffn": F, "experts": E},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
                            "sample": f"{sample} tokens per step of the {name} layer"},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    from paper_2305_13525_b200 import MOE_F_NVLS, MOE_F_STATS, MOE_F_TIMING, MoEConfig, MoELayer, lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    lib()  # fail loudly if the CUDA library is missing

    name, T, H, F, E, gt, gep = workload(args, world)
    dtd = not args.vanilla
    cfg = MoEConfig(T, H, F, E, 1.0, gt, gep, dtd, MOE_F_STATS | MOE_F_TIMING | (MOE_F_NVLS if args.nvls else 0))
    layer = MoELayer(cfg, world, rank, dev)
    L = layer.layout
    El, Fl = L["experts_local"], L["ffn_local"]
    group = L["d"] * gep + L["ep"]

    def gen(shape, seed, scale=1.0, dtype=torch.bfloat16):
        g = torch.Generator(device=dev).manual_seed(seed)
        return (torch.randn(shape, generator=g, device=dev) * scale).to(dtype)

    x = gen((T, H), BASE_SEED + group)
    dy = gen((T, H), BASE_SEED + 3000 + group)
    wg = gen((H, E), BASE_SEED + 1000, 1 / math.sqrt(H), torch.float32)
    w1 = gen((El, Fl, H), BASE_SEED + 2000 + rank, 1 / math.sqrt(H))
    w2 = gen((El, H, Fl), BASE_SEED + 5000 + rank, 1 / math.sqrt(F))
    y = torch.empty_like(x)
    saved = layer.new_saved()
    grads = (torch.empty_like(x), torch.empty_like(wg), torch.empty_like(w1), torch.empty_like(w2))
    stream = torch.cuda.current_stream()

    def step():
        layer.moe_forward(x, wg, w1, w2, y=y, saved=saved)
        layer.moe_backward(dy, saved, x, wg, w1, w2, out=grads)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    layer.moe_stats()          # resolve warm-up events
    layer.moe_stats_reset()
    # throughput pass: no per-class events between the kernels (they would break the
    # programmatic-dependent-launch overlap of consecutive kernels); the per-class
    # breakdown and the roofline come from a second, instrumented pass of the same steps
    layer.moe_set_timing(False)
    clocks = ClockSampler(local)
    clocks.start()
    nvl = NvlinkCounter(local) if world > 1 else None
    time.sleep(0.3)
    barrier()
    nvl_a = nvl.read() if nvl else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    for i in range(args.steps):
        marks[i].record(stream)
        step()
    marks[args.steps].record(stream)
    e1.record(stream)
    barrier()
    nvl_b = nvl.read() if nvl else None
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    ms_median = float(np.median(step_ms))
    st_a = layer.moe_stats()   # ledger / launches of the throughput pass
    # instrumented pass: CUDA events around every kernel class, on the launching streams
    layer.moe_set_timing(True)
    layer.moe_stats_reset()
    barrier()
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    for i in range(args.steps):
        step()
    i1.record(stream)
    barrier()
    ms_instr = i0.elapsed_time(i1) / args.steps
    st = layer.moe_stats()
    st["kernel_launches"] = st_a["kernel_launches"]
    ms_t = torch.tensor([ms], device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    S = world // gt
    tokens_per_step = S * T
    value = tokens_per_step / (ms_max / 1e3)

    # ---- roofline of the dominant kernel class: the tcgen05 expert GEMMs
    rt = layer.moe_routing(saved)
    kept_local = int(rt["count"].sum().item())  # this group's kept tokens
    kept_t = torch.tensor([kept_local], device=dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(kept_t)
    kept_all = float(kept_t.item()) / gt  # kept tokens over all token groups (TP ranks duplicate)
    # algorithmic GEMM FLOPs per rank per step: 12 * H * F_l per kept token routed to this rank's
    # experts; on average kept_all / G_ep tokens reach each EP rank (every TP rank holds F/G_t).
    gemm_flops_step = 12.0 * H * Fl * kept_all / gep
    gemm_ms = st["kernel_ms"]["gemm"] / args.steps
    peaks, peak_src = load_peaks()
    achieved = gemm_flops_step / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    # the GEMMs are timed inside a long step (back-to-back launches under the power cap), so
    # the denominator is the measured SUSTAINED bf16 figure (the contract's rule for a kernel
    # timed inside a long step); the burst fraction is reported beside it, the same in every line
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == name:
            traffic = tj["dram_bytes_per_launch"]
    except Exception:
        pass
    launches_per_step = sum(st["kernel_launches"].values()) / args.steps
    gemm_launch_ms = gemm_ms / 6.0
    roofline = {"bound": "tensor", "kernel": "gemm2_kernel (tcgen05 cta_group::2, 6 launches/step)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "peak_kind": f"{peak_src} bf16 sustained (GEMMs timed inside the step)",
                "peak_burst": peaks["bf16_tflops"],
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "frac_of_burst": (achieved / peaks["bf16_tflops"]) if achieved else None,
                "algorithmic_flop_per_launch": gemm_flops_step / 6.0,
                # padded: every capacity slot computed (empty slots included), SURVEY §8(d)
                "padded_tflops": (12.0 * H * Fl * El * L["rows_per_expert"]) / (gemm_ms / 1e3) / 1e12
                if gemm_ms > 0 else None,
                "frac_of_vendor_2250": (achieved / 2250.0) if achieved else None,
                "ms_per_launch": gemm_launch_ms, "share_of_step": gemm_ms / ms_instr}
    per_class = {k: v / args.steps for k, v in st["kernel_ms"].items()}
    # HBM-bound steps: algorithmic bytes per step / measured time; slices of the
    # slot space this rank dispatches: DTD -> 1 of G_t, vanilla / G_t = 1 -> all
    C = L["capacity"]
    slot_rows = E * C // (gt if (dtd and gt > 1) else 1)
    kept_group = kept_local
    row = H * 2
    hbm_bytes = {"route": T * row + T * E * 4,                          # F1+F2: read x, write logits
                 "dispatch": 2 * slot_rows * row,                       # read x row, write slot row
                 "combine": 2 * T * row,                                # read O row, write y row
                 "combine_bwd": 2 * T * row + slot_rows * row}          # read dy + O, write dO
    if world == 1:
        # one GPU: F11 is fused into F7's epilogue (dropped rows are zeroed by the dispatch
        # launch), so it has no separate HBM figure; the combine-backward launch also
        # writes dl [T][E] fp32 and the K-extension rows [E*C][64] bf16
        hbm_bytes.pop("combine")
        hbm_bytes["combine_bwd"] += T * E * 4 * 2 + slot_rows * 128
    hbm = {}
    for k, b in hbm_bytes.items():
        t_ms = per_class.get(k, 0.0)
        if t_ms > 0:
            gbs = b / (t_ms / 1e3) / 1e9
            hbm[k] = {"bytes": b, "ms": t_ms, "GB/s": gbs, "frac": gbs / peaks["hbm_gbs"]}
    if world == 1:
        hbm["combine"] = "fused into the F7 GEMM epilogue (EPI_COMBINE); dropped rows zeroed by the dispatch launch"
    if "route" in hbm:
        # the gate also has a compute roofline: 2*H*E flop per token (x . Wg); on the tensor
        # cores with Wg split in three bf16 terms (3x the flops) it is far from that bound,
        # so HBM (streaming x) is the roofline that binds; the FP32-ALU figure is what the
        # contraction would need on CUDA cores
        r_ms = hbm["route"]["ms"]
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12   # TFLOP/s: SMs x FP32 lanes x FMA x max clock
        hbm["route"]["flop"] = 2.0 * T * H * E
        hbm["route"]["fp32_alu_frac"] = (2.0 * T * H * E / (r_ms / 1e3) / 1e12) / fp32_peak
    del kept_group

    # ---- e2e through the public API with host buffers (pinned). Every step copies its
    # inputs host->device and its results device->host inside the timed region; the
    # copies run on a second stream, double-buffered, so step i's transfers overlap
    # step i-1's / i+1's compute (what a training loop feeding the layer would do).
    e2e = None
    layer.moe_set_timing(False)
    if not args.no_e2e:
        nbuf = 2
        hx = [torch.empty_like(x, device="cpu").pin_memory().copy_(x) for _ in range(nbuf)]
        hdy = [torch.empty_like(dy, device="cpu").pin_memory().copy_(dy) for _ in range(nbuf)]
        hy = [torch.empty_like(y, device="cpu").pin_memory() for _ in range(nbuf)]
        hdx = [torch.empty_like(x, device="cpu").pin_memory() for _ in range(nbuf)]
        xd = [torch.empty_like(x) for _ in range(nbuf)]
        dyd = [torch.empty_like(dy) for _ in range(nbuf)]
        yd = [torch.empty_like(y) for _ in range(nbuf)]
        gd = [(torch.empty_like(x), torch.empty_like(wg), torch.empty_like(w1), torch.empty_like(w2))
              for _ in range(nbuf)]
        sv = [layer.new_saved() for _ in range(nbuf)]
        hs = torch.cuda.Stream(device=dev)   # host -> device
        ds = torch.cuda.Stream(device=dev)   # device -> host
        h2d_done = [torch.cuda.Event() for _ in range(nbuf)]
        comp_done = [torch.cuda.Event() for _ in range(nbuf)]
        d2h_done = [torch.cuda.Event() for _ in range(nbuf)]

        def e2e_run(n):
            def h2d(i):
                k = i % nbuf
                with torch.cuda.stream(hs):
                    if i >= nbuf:
                        hs.wait_event(comp_done[k])   # buffer k's previous compute finished
                    xd[k].copy_(hx[k], non_blocking=True)
                    dyd[k].copy_(hdy[k], non_blocking=True)
                    h2d_done[k].record(hs)
            h2d(0)
            for i in range(n):
                k = i % nbuf
                if i + 1 < n:
                    h2d(i + 1)                         # next step's inputs in flight
                stream.wait_event(h2d_done[k])
                if i >= nbuf:
                    stream.wait_event(d2h_done[k])    # buffer k's previous results read back
                layer.moe_forward(xd[k], wg, w1, w2, y=yd[k], saved=sv[k])
                layer.moe_backward(dyd[k], sv[k], xd[k], wg, w1, w2, out=gd[k])
                comp_done[k].record(stream)
                with torch.cuda.stream(ds):
                    ds.wait_event(comp_done[k])
                    hy[k].copy_(yd[k], non_blocking=True)
                    hdx[k].copy_(gd[k][0], non_blocking=True)
                    d2h_done[k].record(ds)
            stream.wait_stream(hs)
            stream.wait_stream(ds)

        e2e_run(3)
        barrier()
        n_e2e = max(6, min(args.steps, 30))
        e0.record(stream)
        e2e_run(n_e2e)
        e1.record(stream)
        barrier()
        ms_e = torch.tensor([e0.elapsed_time(e1) / n_e2e], device=dev)
        if dist is not None:
            dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
        nb = x.numel() * 2
        e2e = {"value": tokens_per_step / (float(ms_e.item()) / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb,
               "ms_per_step": float(ms_e.item()),
               "what": "pinned host x, dy -> device; moe_forward + moe_backward; y, dx -> host; "
                       "H2D / D2H on their own streams, double-buffered (next step's H2D overlaps this step's compute)"}

    optim = None
    if not args.no_optim:
        optim = measure_optimizer(grads[2], grads[3], peaks, args.steps, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(H, F, E)

    if rank == 0:
        out = {"metric": "MoE-layer fwd+bwd tokens/s", "value": value, "unit": "tokens/s",
               "value_per_gpu": value / world,
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
               "ms_per_step_median": ms_median,
               "ms_per_step_instrumented": ms_instr,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (x, dy ~ N(0,1); Wg ~ N(0,1/H); W1 ~ N(0,1/H); W2 ~ N(0,1/F))",
               "config": {"workload": name, "tokens_per_group": T, "hidden": H, "ffn": F, "experts": E,
                          "capacity_factor": 1.0, "g_tensor": gt, "g_expert": gep,
                          "dtd": bool(dtd and gt > 1), "nvls": bool(args.nvls and dtd and gt > 1), "token_groups": S,
                          "l2": "no flush: >1 GB expert weights + activations per step exceed 126 MB L2"},
               "roofline": roofline, "hbm_steps": hbm, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(round(launches_per_step * args.steps)),
               "launches_per_step": launches_per_step, "clocks": clk,
               "kernel_ms_per_step": per_class,
               "dropped_tokens": st["dropped_tokens"], "tie_tokens": st["tie_tokens"],
               "collectives": {"calls": st["calls"], "wire_bytes": st["wire_bytes"]},
               "optimizer": optim}
        if world > 1:
            # a2a bandwidth: bytes this rank sends to other ranks per step. In peer
            # mode with G_t = 1 the dispatch direction (X forward, dO backward: half of the a2a
            # bytes) travels on the copy engines (class "xfer", CUDA events on the side stream
            # around the copies, overlapped with the GEMMs) and the return direction is stored by
            # the GEMM epilogues themselves (F7+F9, B5+B8), so the link rate is the dispatch
            # bytes / xfer time; otherwise (fused SM stores / NCCL) the time basis is the kernel
            # classes that move the bytes, a lower bound.
            wb = {k: v / args.steps for k, v in st["wire_bytes"].items()}
            egress = sum(wb.values())
            xfer_ms = per_class.get("xfer", 0.0)
            fused_return = os.environ.get("MOE_NO_FUSED_RETURN", "0") != "1"
            if xfer_ms > 0 and gt == 1:
                ex_ms = xfer_ms
                if fused_return:
                    egress_rate = wb["a2a"] / 2
                    basis = "dispatch-direction copy-engine transfers (xfer class) for half the a2a bytes; " \
                            "the return half is stored by the GEMM epilogues"
                else:
                    egress_rate = egress
                    basis = "copy-engine transfers (xfer class, side stream)"
                gbs = egress_rate / (ex_ms / 1e3) / 1e9
            else:
                ex_ms = per_class["comm"] + per_class["dispatch"] + per_class["combine_bwd"] + xfer_ms
                basis = "comm + dispatch + combine_bwd + xfer classes (lower bound)"
                gbs = egress / (ex_ms / 1e3) / 1e9 if ex_ms > 0 else None
            out["comm_ms_per_step"] = per_class["comm"]
            out["a2a"] = {"a2a_bytes_per_step": wb["a2a"], "egress_bytes_per_step": egress,
                          "transfer_ms_per_step": ex_ms, "egress_GB/s": gbs,
                          "peak_GB/s": 770.0, "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                          "frac": gbs / 770.0 if gbs else None, "time_basis": basis,
                          "exposed_comm_ms_per_step": per_class["comm"],
                          "nvlink_rank0": nvl.delta(nvl_a, nvl_b, args.steps) if nvl else None}
        print(json.dumps(out), flush=True)
    layer.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
