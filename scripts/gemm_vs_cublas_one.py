"""One launch each of our GEMM (ee_test_gemm) and cuBLAS (torch.mm) on the a2
shape (65536 x 57344 x 8192, both operands K-major), for an ncu --set full
comparison (DRAM bytes, L2 hit rate, tensor-pipe activity, cuBLAS's kernel
name = its tile / cluster choice)."""
import os
import sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2402_00518_b200 as ee

ee.load()
M, N, K = 65536, 57344, 8192
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.randn(M, K, generator=g, device="cuda") * 0.02).bfloat16()
B = (torch.randn(N, K, generator=g, device="cuda") * 0.02).bfloat16()
C = torch.empty(M, N, device="cuda")
Cb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    ee.ee_test_gemm(A, B, C, True, True, M, N, K)
    torch.mm(A, B.t(), out=Cb)
torch.cuda.synchronize()
print("ok")
