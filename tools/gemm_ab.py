"""A/B of GEMM kernel variants selected by the MOE_GEMM_DBG environment knob.

Interleaves the variants case by case and repeats the sweep, reporting the
minimum time per (case, variant), so slow power-state drift hits all variants.

    python tools/gemm_ab.py --dbg 0 4 --reps 5
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
    ap.add_argument("--dbg", type=int, nargs="+", default=[0, 4])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    sh = synth.CONFIGS[a.config]
    El, Fl, H = sh.experts // sh.g_expert, sh.ffn // sh.g_tensor, sh.hidden
    R = sh.g_expert * -(-sh.tokens // sh.experts)
    bf = torch.bfloat16
    X = torch.randn(El, R, H, device="cuda", dtype=bf)
    W1 = torch.randn(El, Fl, H, device="cuda", dtype=bf) * 0.02
    W2 = torch.randn(El, H, Fl, device="cuda", dtype=bf) * 0.02
    Hp = torch.empty(El, R, Fl, device="cuda", dtype=bf)
    A = torch.empty(El, R, Fl, device="cuda", dtype=bf)
    Y = torch.empty(El, R, H, device="cuda", dtype=bf)
    dW1, dW2 = torch.empty_like(W1), torch.empty_like(W2)
    cases = {"F6 gelu": (X, W1, Hp, 0, 0, 1, A), "F7": (A, W2, Y, 0, 0, 0, None),
             "B4 dgelu": (Y, W2, A, 0, 1, 2, Hp), "B5": (A, W1, X, 0, 1, 0, None),
             "B6 dW2": (Y, A, dW2, 1, 1, 0, None), "B6 dW1": (A, X, dW1, 1, 1, 0, None)}
    best = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.reps):
        for name, (Aop, Bop, D, amn, bmn, epi, aux) in cases.items():
            for d in a.dbg:
                os.environ["MOE_GEMM_DBG"] = str(d)
                for _ in range(2):
                    moe_gemm_bf16(Aop, Bop, D, amn, bmn, epi, aux, 0)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(a.iters):
                    moe_gemm_bf16(Aop, Bop, D, amn, bmn, epi, aux, 0)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                k = (name, d)
                best[k] = min(best.get(k, 1e9), ms)
    out = {name: {str(d): round(best[(name, d)] * 1e3, 1) for d in a.dbg} for name in cases}
    out["total_us"] = {str(d): round(sum(best[(n, d)] for n in cases) * 1e3, 1) for d in a.dbg}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
