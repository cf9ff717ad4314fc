"""Small attention forward + backward (both forward kernels) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2402_00518_b200 as ee
ee.load()
B, T, Hq, Hkv = 1, 384, 2, 1
n = B * T
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
k = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
o = torch.empty_like(q); lse2 = torch.empty(n, Hq, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
scr = torch.empty(n, Hq, device="cuda")
for impl in (1, 2):
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr, impl=impl)
torch.cuda.synchronize()
print("ok")
