"""Same-box A/B of the expert GEMMs of two builds of libmoe.so (development tool).

    python tools/gemm_ab.py LIB_A LIB_B [--reps 5] [--iters 10] [--config 1.3b]

Loads both libraries with ctypes (only moe_gemm_bf16, whose ABI is unchanged across
rounds) and times the F6 / F7 / B4 / B5 / B6 shapes of one layer step on the same
tensors, interleaving A and B per repetition so box clocks and the power cap hit both.
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13525_b200 import synth  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    I, P = ctypes.c_int, ctypes.c_void_p
    L.moe_gemm_bf16.argtypes = [I, I, I, I, P, I, P, I, P, I, P, I, P]
    L.moe_gemm_bf16.restype = I
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--config", default="1.3b")
    a = ap.parse_args()
    libs = [load(p) for p in a.libs]
    sh = synth.CONFIGS[a.config]
    El, Fl, H = sh.experts // sh.g_expert, sh.ffn // sh.g_tensor, sh.hidden
    R = sh.g_expert * -(-sh.tokens // sh.experts)
    bf = torch.bfloat16
    dev = "cuda"
    X = torch.randn(El, R, H, device=dev, dtype=bf)
    W1 = torch.randn(El, Fl, H, device=dev, dtype=bf) * 0.02
    W2 = torch.randn(El, H, Fl, device=dev, dtype=bf) * 0.02
    Hp = torch.randn(El, R, Fl, device=dev, dtype=bf)
    A = torch.randn(El, R, Fl, device=dev, dtype=bf)
    Y = torch.randn(El, R, H, device=dev, dtype=bf)
    dW1, dW2 = torch.empty_like(W1), torch.empty_like(W2)
    cases = {
        "F6 gelu": (X, W1, Hp, 0, 0, 1, A),
        "F7": (A, W2, Y, 0, 0, 0, None),
        "B4 dgelu": (Y, W2, A, 0, 1, 2, Hp),
        "B5": (A, W1, X, 0, 1, 0, None),
        "B6 dW2": (Y, A, dW2, 1, 1, 0, None),
        "B6 dW1": (A, X, dW1, 1, 1, 0, None),
    }
    stream = torch.cuda.current_stream().cuda_stream

    def call(L, c):
        Aop, Bop, D, amn, bmn, epi, aux = c
        M, N = D.shape[1], D.shape[2]
        K = Aop.shape[1] if amn else Aop.shape[2]
        r = L.moe_gemm_bf16(El, M, N, K, Aop.data_ptr(), amn, Bop.data_ptr(), bmn, D.data_ptr(), epi,
                            aux.data_ptr() if aux is not None else None, 0, stream)
        assert r == 0, r

    res = {n: [[], []] for n in cases}
    tot = [[], []]
    for _ in range(a.reps):
        for li, L in enumerate(libs):
            for c in cases.values():
                call(L, c)
            t = 0.0
            for n, c in cases.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    call(L, c)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                res[n][li].append(ms)
                t += ms
            tot[li].append(t)
    out = {n: {"A_ms": round(min(v[0]), 4), "B_ms": round(min(v[1]), 4)} for n, v in res.items()}
    out["total"] = {"A_ms": round(min(tot[0]), 4), "B_ms": round(min(tot[1]), 4),
                    "A_all": [round(x, 3) for x in tot[0]], "B_all": [round(x, 3) for x in tot[1]]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
