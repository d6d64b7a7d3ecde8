"""cuBLAS (torch.bmm) on the 1.3B layer's six expert-GEMM shapes, for comparison with
gemm2_kernel (development tool; same operand majors as the layer's GEMMs).

    python tools/cublas_ref.py
"""
import torch

E, R, H, F = 16, 1024, 2048, 8192
dev = "cuda"


def bench(fn, flops, name, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(it):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{name:40s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s")


def r(*s):
    return torch.randn(*s, device=dev, dtype=torch.bfloat16)


X, W1, W2 = r(E, R, H), r(E, F, H), r(E, H, F)
A, dY, dH = r(E, R, F), r(E, R, H), r(E, R, F)
fl = 2.0 * E * R * H * F
bench(lambda: torch.bmm(X, W1.transpose(1, 2)), fl, "F6  X W1^T      [R,H]x[H,F]")
bench(lambda: torch.bmm(A, W2.transpose(1, 2)), fl, "F7  A W2^T      [R,F]x[F,H]")
bench(lambda: torch.bmm(dY, W2), fl, "B4  dY W2       [R,H]x[H,F]")
bench(lambda: torch.bmm(dH, W1), fl, "B5  dH W1       [R,F]x[F,H]")
bench(lambda: torch.bmm(dY.transpose(1, 2), A), fl, "B6  dY^T A      [H,R]x[R,F]")
bench(lambda: torch.bmm(dH.transpose(1, 2), X), fl, "B6' dH^T X      [F,R]x[R,H]")
M = 8192
P, Q = r(M, M), r(M, M)
bench(lambda: P @ Q, 2.0 * M ** 3, "8192^3 (MEASURED_PEAKS burst shape)")
