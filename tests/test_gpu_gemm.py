"""The tcgen05 expert GEMM (moe_gemm_bf16) against a plain PyTorch fp32 reference."""
import pytest
import torch

from paper_2305_13525_b200 import moe_gemm_bf16

pytestmark = pytest.mark.gpu


def _ref(A, B, a_mn, b_mn, epi, aux):
    Af = A.float()
    Bf = B.float()
    if a_mn:
        Af = Af.transpose(1, 2)  # [b][K][M] -> [b][M][K]
    if not b_mn:
        Bf = Bf.transpose(1, 2)  # [b][N][K] -> [b][K][N]
    acc = torch.bmm(Af, Bf)
    if epi == 2:
        acc = acc * aux.float()
    return acc


def _gelu_grad(h):
    k = 0.7978845608028654
    th = torch.tanh(k * (h + 0.044715 * h ** 3))
    return 0.5 * (1 + th) + 0.5 * h * (1 - th * th) * k * (1 + 3 * 0.044715 * h * h)


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


COMBOS = [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 2), (1, 1, 0)]
SHAPES = [(2, 200, 320, 136), (1, 128, 256, 64), (3, 64, 64, 8), (1, 1024, 1024, 2048)]


@pytest.mark.parametrize("a_mn,b_mn,epi", COMBOS)
@pytest.mark.parametrize("batch,M,N,K", SHAPES)
@pytest.mark.parametrize("impl", [0, 1])
def test_gemm_vs_torch(a_mn, b_mn, epi, batch, M, N, K, impl):
    g = torch.Generator(device="cuda").manual_seed(1234 + M + N + K)
    dev = "cuda"
    A = torch.randn((batch, K, M) if a_mn else (batch, M, K), generator=g, device=dev).bfloat16()
    B = torch.randn((batch, K, N) if b_mn else (batch, N, K), generator=g, device=dev).bfloat16()
    D = torch.full((batch, M, N), float("nan"), device=dev, dtype=torch.bfloat16)
    aux = None
    if epi == 1:
        aux = torch.full((batch, M, N), float("nan"), device=dev, dtype=torch.bfloat16)
    elif epi == 2:
        aux = torch.randn((batch, M, N), generator=g, device=dev).bfloat16()
    moe_gemm_bf16(A, B, D, a_mn, b_mn, epi, aux, impl)
    torch.cuda.synchronize()
    ref = _ref(A, B, a_mn, b_mn, epi, aux)
    assert torch.isfinite(D.float()).all()
    if epi == 1:
        assert _rel(D, _gelu_grad(ref)) < 1e-2
        gelu = torch.nn.functional.gelu(ref, approximate="tanh")
        assert torch.isfinite(aux.float()).all()
        assert _rel(aux, gelu) < 1e-2
    else:
        assert _rel(D, ref) < 5e-3


def test_gemm_tc_matches_simt_reference_large():
    """The tcgen05 kernel and the SIMT cross-check agree on a multi-wave problem."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(7)
    A = torch.randn(4, 1024, 2048, generator=g, device=dev).bfloat16()
    B = torch.randn(4, 2048, 2048, generator=g, device=dev).bfloat16()
    D0 = torch.empty(4, 1024, 2048, device=dev, dtype=torch.bfloat16)
    D1 = torch.empty_like(D0)
    moe_gemm_bf16(A, B, D0, 0, 0, 0, None, 0)
    moe_gemm_bf16(A, B, D1, 0, 0, 0, None, 1)
    torch.cuda.synchronize()
    assert _rel(D0, D1) < 5e-3
