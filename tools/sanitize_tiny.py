"""compute-sanitizer driver: one forward + backward of every kernel family on
tiny shapes, one GPU, plus an emulated 2 x 2 (G_t, G_ep) group (the peer-exchange
kernels). No oracle — the sanitizer report is the result.

    compute-sanitizer --tool memcheck  python tools/sanitize_tiny.py
    compute-sanitizer --tool racecheck python tools/sanitize_tiny.py --no-emu
    compute-sanitizer --tool synccheck python tools/sanitize_tiny.py --no-emu
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_13525_b200 import (MOE_F_AUX_LOSS, MOE_F_CAC, MOE_F_CHECKPOINT, MOE_F_RANDOM_PRIORITY,  # noqa: E402
                                   MoEConfig, MoELayer, moe_adamw_step, synth)


def t16(a, dev):
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)


def one(T, H, F, E, flags=0, top_k=1, replay=False):
    dev = torch.device("cuda", 0)
    shape = synth.LayerShape("san", T, H, F, E)
    x, dy = t16(synth.make_x(shape), dev), t16(synth.make_dy(shape), dev)
    wg = torch.from_numpy(synth.make_wg(shape)).to(dev)
    w1b, w2b = synth.make_experts(shape)
    w1, w2 = t16(w1b, dev), t16(w2b, dev)
    layer = MoELayer(MoEConfig(T, H, F, E, 1.0, 1, 1, True, 1 | flags, top_k=top_k), 1, 0, dev)
    y, saved = layer.moe_forward(x, wg, w1, w2)
    if replay:
        layer.moe_forward_replay(saved, x, wg, w1, w2)
    dx, dwg, dw1, dw2 = layer.moe_backward(dy, saved, x, wg, w1, w2)
    torch.cuda.synchronize()
    layer.close()
    return dw1


def main():
    cases = [dict(T=300, H=128, F=192, E=5), dict(T=256, H=256, F=256, E=16), dict(T=200, H=128, F=128, E=32),
             dict(T=256, H=128, F=128, E=8, flags=MOE_F_AUX_LOSS | MOE_F_RANDOM_PRIORITY),
             dict(T=256, H=128, F=128, E=8, top_k=2),
             dict(T=256, H=128, F=128, E=8, flags=MOE_F_CHECKPOINT | MOE_F_CAC, replay=True)]
    for c in cases:
        dw1 = one(**c)
        print("ok", c, flush=True)
    g = dw1.reshape(-1)
    n = g.numel()
    p, m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    moe_adamw_step(g, p, m, v, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, step=1)
    torch.cuda.synchronize()
    print("ok optimizer", flush=True)
    if "--no-emu" not in sys.argv:
        from tests import emu
        shape = synth.LayerShape("san-emu", 256, 128, 256, 8, 1.0, 2, 2)
        wl = emu.Workload(shape)
        emu.run_modes(wl, {"dtd": wl.config(True), "van": wl.config(False)})
        print("ok emulated tp2ep2", flush=True)


if __name__ == "__main__":
    main()
