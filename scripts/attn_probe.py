"""Standalone launch of the attention kernels at the 13b_layer shape (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2402_00518_b200 as ee

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bwd = len(sys.argv) > 2 and sys.argv[2] == "bwd"
T, Hq, Hkv, B = 2048, 40, 40, 16
n = B * T
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn(n, Hq * 128, device="cuda", generator=g)).bfloat16()
k = (torch.randn(n, Hkv * 128, device="cuda", generator=g)).bfloat16()
v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
o = torch.empty_like(q)
lse2 = torch.empty(n, Hq, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
scr = torch.empty(n, Hq, device="cuda")
kw = dict(dout=do, dq=dq, dk=dk, dv=dv, scratch=scr) if bwd else {}
for _ in range(3):
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl, **kw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl, **kw)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
fl = 2 * 2 * 128 * Hq * n * (T + 1) / 2 * (3 if bwd else 1)
print(f"impl={impl} bwd={bwd} {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s (algorithmic fwd{'+bwd' if bwd else ''})")
