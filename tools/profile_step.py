"""One (or a few) MoE-layer fwd+bwd steps at a BASELINE shape, for ncu captures.

    python tools/profile_step.py [--config 1.3b] [--steps 1] [--tokens T]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13525_b200 import MoEConfig, MoELayer, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1.3b")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=None)
    a = ap.parse_args()
    shape = synth.CONFIGS[a.config]
    T = a.tokens or shape.tokens
    dev = torch.device("cuda", 0)
    layer = MoELayer(MoEConfig(T, shape.hidden, shape.ffn, shape.experts), 1, 0, dev)
    g = torch.Generator(device=dev).manual_seed(0)
    H, F, E = shape.hidden, shape.ffn, shape.experts
    x = torch.randn(T, H, generator=g, device=dev).bfloat16()
    dy = torch.randn(T, H, generator=g, device=dev).bfloat16()
    wg = torch.randn(H, E, generator=g, device=dev) / math.sqrt(H)
    w1 = (torch.randn(E, F, H, generator=g, device=dev) / math.sqrt(H)).bfloat16()
    w2 = (torch.randn(E, H, F, generator=g, device=dev) / math.sqrt(F)).bfloat16()
    for _ in range(a.steps):
        y, saved = layer.moe_forward(x, wg, w1, w2)
        layer.moe_backward(dy, saved, x, wg, w1, w2)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
