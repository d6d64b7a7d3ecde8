"""Development tool: the multi-GPU product path of one (G_t, G_ep) layout on ONE GPU through
emulated ranks (tests/emu.py), for per-kernel launch lists under ncu:

    ncu --metrics gpu__time_duration.sum --csv python tools/emu_step.py --config 1.3b --gep 2 --steps 2

Every rank runs `steps` forward+backward passes on seeded synthetic inputs (no oracle).
"""
import argparse
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13525_b200 import synth  # noqa: E402
from tests.emu import Workload, fwd_bwd, run_modes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1.3b")
    ap.add_argument("--gt", type=int, default=1)
    ap.add_argument("--gep", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--vanilla", action="store_true")
    a = ap.parse_args()
    sh = dataclasses.replace(synth.CONFIGS[a.config], g_tensor=a.gt, g_expert=a.gep)
    wl = Workload(sh, tokens=a.tokens)

    def sched(layer, inp, st):
        for _ in range(a.steps):
            out = fwd_bwd(layer, inp, st)
        return out["stats"]

    res = run_modes(wl, {"m": wl.config(dtd=not a.vanilla)}, schedule=sched)
    torch.cuda.synchronize()
    print("ok", a.config, "gt", a.gt, "gep", a.gep, "launches", res[0]["m"]["kernel_launches"])


if __name__ == "__main__":
    main()
