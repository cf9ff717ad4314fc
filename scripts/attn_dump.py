"""Attention forward + backward at a ragged causal shape (T = 192, GQA 2:1) and
the 13B Layer shape; saves o / dq / dk / dv so two library builds can be
compared bitwise (EE_LIB_AB = the .so to load).  Usage: attn_dump.py OUT.pt"""
import os
import sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2402_00518_b200 as ee

ee.load(os.environ.get("EE_LIB_AB", ee.LIB_PATH))
out = {}
for (B, T, Hq, Hkv) in [(2, 192, 4, 2), (4, 2048, 40, 40)]:
    n = B * T
    g = torch.Generator(device="cuda").manual_seed(7)
    q = (torch.randn(n, Hq * 128, device="cuda", generator=g) * 2).bfloat16()
    k = (torch.randn(n, Hkv * 128, device="cuda", generator=g) * 2).bfloat16()
    v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
    o = torch.empty_like(q)
    lse2 = torch.empty(n, Hq, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    scr = torch.empty(n, Hq, device="cuda")
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr,
                         impl=2)
    torch.cuda.synchronize()
    out[f"T{T}"] = {"o": o.cpu(), "dq": dq.cpu(), "dk": dk.cpu(), "dv": dv.cpu()}
torch.save(out, sys.argv[1])
print("saved", sys.argv[1])
