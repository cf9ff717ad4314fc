"""Attention backward timing at the Layer-exit shapes (ee_test_attention with
dout; forward excluded by subtracting a forward-only run)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2402_00518_b200 as ee
ee.load(os.environ.get("EE_LIB_AB", ee.LIB_PATH))
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

    def t(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    fwd = t(lambda: ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=2))
    both = t(lambda: ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk,
                                          dv=dv, scratch=scr, impl=2))
    bwd = both - fwd
    fl = 4.0 * n * Hq * 128 * (T + 1) / 2 * 2     # dV, dP, dQ, dK over the causal triangle
    print(json.dumps({"shape": f"B{B} T{T} Hq{Hq} Hkv{Hkv}", "fwd_ms": round(fwd, 3),
                      "bwd_ms": round(bwd, 3), "bwd_alg_tflops": round(fl / bwd / 1e9, 1)}),
          flush=True)
