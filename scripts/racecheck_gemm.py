import sys, torch
sys.path.insert(0, ".")
import paper_2402_00518_b200 as ee
M, N, K = 512, 512, 256
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda")
ee.ee_test_gemm(A, B, C, True, True, M, N, K)
torch.cuda.synchronize()
print("max err", (C - A.float() @ B.float().T).abs().max().item())
