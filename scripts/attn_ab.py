"""Attention forward A/B at the Layer-exit shape (13B: 40 heads, T = 2048, 16
sequences): one-tile vs two-tile tcgen05 forward, CUDA-event timed, plus the
backward for reference.  TFLOP/s on the causal algorithmic count
2 * 2 * n * h * (T + 1) / 2 (QK^T and PV over the lower triangle)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2402_00518_b200 as ee
ee.load()
for (B, T, Hq, Hkv) in [(16, 2048, 40, 40), (16, 2048, 64, 8)]:
    n = B * T
    g = torch.Generator(device="cuda").manual_seed(1)
    q = (torch.randn(n, Hq * 128, device="cuda", generator=g) * 2).bfloat16()
    k = (torch.randn(n, Hkv * 128, device="cuda", generator=g) * 2).bfloat16()
    v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
    o = torch.empty_like(q); lse2 = torch.empty(n, Hq, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    scr = torch.empty(n, Hq, device="cuda")
    fl = 2.0 * 2 * n * Hq * 128 * (T + 1) / 2
    res = {"shape": f"B{B} T{T} Hq{Hq} Hkv{Hkv}"}
    for impl in (1, 2, 1, 2):
        for _ in range(3):
            ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.setdefault(f"fwd_impl{impl}", []).append({"ms": round(ms, 3), "tflops": round(fl / ms / 1e9, 1)})
    for _ in range(2):
        ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr, impl=2)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr, impl=2)
    e1.record(); torch.cuda.synchronize()
    res["fwd_plus_bwd_impl2_ms"] = round(e0.elapsed_time(e1) / 5, 3)
    print(json.dumps(res), flush=True)
