"""Times the six expert GEMMs of one layer step in isolation (CUDA events, L2-cold-ish).

    python tools/gemm_bench.py [--config 1.3b] [--impl 0 2] [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13525_b200 import moe_gemm_bf16, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1.3b")
    ap.add_argument("--impl", type=int, nargs="+", default=[0])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    sh = synth.CONFIGS[a.config]
    El = sh.experts // sh.g_expert
    Fl = sh.ffn // sh.g_tensor
    R = sh.g_expert * -(-sh.tokens // sh.experts)
    H = sh.hidden
    dev = "cuda"
    bf = torch.bfloat16
    X = torch.randn(El, R, H, device=dev, dtype=bf)
    W1 = torch.randn(El, Fl, H, device=dev, dtype=bf) * 0.02
    W2 = torch.randn(El, H, Fl, device=dev, dtype=bf) * 0.02
    Hp = torch.empty(El, R, Fl, device=dev, dtype=bf)
    A = torch.empty(El, R, Fl, device=dev, dtype=bf)
    Y = torch.empty(El, R, H, device=dev, dtype=bf)
    dW1 = torch.empty_like(W1)
    dW2 = torch.empty_like(W2)
    cases = {
        "F6 X.W1^T+gelu": (X, W1, Hp, 0, 0, 1, A),
        "F6-shape plain": (X, W1, Hp, 0, 0, 0, None),
        "F7 A.W2^T": (A, W2, Y, 0, 0, 0, None),
        "B4 dY.W2*gelu'": (Y, W2, A, 0, 1, 2, Hp),
        "B4-shape plain": (Y, W2, A, 0, 1, 0, None),
        "B5 dH.W1": (A, W1, X, 0, 1, 0, None),
        "B6 dY^T.A": (Y, A, dW2, 1, 1, 0, None),
        "B6 dH^T.X": (A, X, dW1, 1, 1, 0, None),
    }
    out = {}
    for impl in a.impl:
        tot = 0.0
        for name, (Aop, Bop, D, amn, bmn, epi, aux) in cases.items():
            Mm, Nn = D.shape[1], D.shape[2]
            K = Aop.shape[1] if amn else Aop.shape[2]
            flops = 2.0 * El * Mm * Nn * K
            for _ in range(a.warmup):
                moe_gemm_bf16(Aop, Bop, D, amn, bmn, epi, aux, impl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                moe_gemm_bf16(Aop, Bop, D, amn, bmn, epi, aux, impl)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            tot += ms
            out[f"impl{impl} {name}"] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1)}
        out[f"impl{impl} total_ms"] = round(tot, 4)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
