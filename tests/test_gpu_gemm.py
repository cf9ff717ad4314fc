"""tcgen05 GEMM kernel vs a plain PyTorch fp32 reference of the same op.

C = A B^T with every combination of operand majorness the step uses (K-major
and MN-major A and B), over shapes spanning several 128x256x64 tiles with
ragged M/N/K tails.  Inputs are bf16; the reference is the fp32 product of the
same bf16 values (torch, CPU), so the only difference is fp32 summation order.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (304, 520, 200), (1000, 264, 1096), (256, 512, 4096), (8, 8, 8)]


@pytest.mark.parametrize("a_kmajor", [True, False])
@pytest.mark.parametrize("b_kmajor", [True, False])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_majors(gpu_lib, a_kmajor, b_kmajor, M, N, K):
    ee = gpu_lib
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    ref = A.float() @ B.float().T
    Ad = (A if a_kmajor else A.T.contiguous()).cuda()
    Bd = (B if b_kmajor else B.T.contiguous()).cuda()
    C = torch.full((M, N), float("nan"), device="cuda")
    ee.ee_test_gemm(Ad, Bd, C, a_kmajor, b_kmajor, M, N, K)
    torch.cuda.synchronize()
    err = (C.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
    # accumulate mode adds onto C
    ee.ee_test_gemm(Ad, Bd, C, a_kmajor, b_kmajor, M, N, K, accumulate=True)
    torch.cuda.synchronize()
    err2 = (C.cpu() - 2 * ref).abs().max().item()
    assert err2 <= 2e-3 * max(1.0, ref.abs().max().item()), err2


def test_gemm_large_k_precision(gpu_lib):
    """K = 16384 (a token-contraction of the weight-gradient GEMMs)."""
    ee = gpu_lib
    g = torch.Generator().manual_seed(1)
    M, N, K = 256, 256, 16384
    A = torch.randn(K, M, generator=g).to(torch.bfloat16)   # MN-major storage
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)
    ref = A.double().T @ B.double()
    C = torch.empty(M, N, device="cuda")
    ee.ee_test_gemm(A.cuda(), B.cuda(), C, False, False, M, N, K)
    torch.cuda.synchronize()
    rel = ((C.cpu().double() - ref).norm() / ref.norm()).item()
    assert rel < 5e-5, rel
