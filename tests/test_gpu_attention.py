"""Causal GQA flash attention kernels (forward + FA2 backward) against a plain
fp32 PyTorch autograd reference of the same op on the same bf16 inputs
(Llama-2 attention; used by the backbone and the Layer exit)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(q, k, v, dout, T, Hq, Hkv):
    n = q.shape[0]
    B = n // T
    qf = q.float().view(B, T, Hq, 128).transpose(1, 2).requires_grad_()
    kf = k.float().view(B, T, Hkv, 128).transpose(1, 2).requires_grad_()
    vf = v.float().view(B, T, Hkv, 128).transpose(1, 2).requires_grad_()
    rep = Hq // Hkv
    kk = kf.repeat_interleave(rep, dim=1)
    vv = vf.repeat_interleave(rep, dim=1)
    s = (qf @ kk.transpose(-1, -2)) / math.sqrt(128)
    mask = torch.ones(T, T, dtype=torch.bool, device=q.device).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)                       # natural log
    o = torch.softmax(s, dim=-1) @ vv
    o.backward(dout.float().view(B, T, Hq, 128).transpose(1, 2))
    flat = lambda t, H: t.transpose(1, 2).reshape(n, H * 128)
    return (flat(o.detach(), Hq), lse.transpose(1, 2).reshape(n, Hq), flat(qf.grad, Hq),
            flat(kf.grad, Hkv), flat(vf.grad, Hkv))


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


@pytest.mark.parametrize("impl", [0, 1, 2], ids=["mma_sync", "tcgen05", "tcgen05_2tile"])
@pytest.mark.parametrize("B,T,Hq,Hkv", [(2, 128, 4, 2), (1, 256, 2, 2), (3, 64, 8, 1),
                                        (1, 512, 4, 1), (2, 192, 2, 1), (1, 2048, 1, 1)])
def test_attention_fwd_bwd_vs_fp32_autograd(gpu_lib, B, T, Hq, Hkv, impl):
    ee = gpu_lib
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + T + Hq)
    n = B * T
    q = (torch.randn(n, Hq * 128, device="cuda", generator=g) * 1.5).bfloat16()
    k = (torch.randn(n, Hkv * 128, device="cuda", generator=g) * 1.5).bfloat16()
    v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
    o = torch.empty_like(q)
    lse2 = torch.empty(n, Hq, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    scr = torch.empty(n, Hq, device="cuda")
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr,
                         impl=impl)
    torch.cuda.synchronize()
    o_r, lse_r, dq_r, dk_r, dv_r = _ref(q, k, v, do, T, Hq, Hkv)
    assert _rel(o, o_r) <= 1e-2
    # lse2 is in log2 units: lse = lse2 * ln 2
    assert torch.allclose(lse2 * math.log(2.0), lse_r, atol=2e-2, rtol=0)
    assert torch.allclose(scr, (do.float() * o.float()).view(n, Hq, 128).sum(-1), rtol=1e-3,
                          atol=1e-3)
    for got, ref, name in ((dq, dq_r, "dq"), (dk, dk_r, "dk"), (dv, dv_r, "dv")):
        assert torch.isfinite(got.float()).all(), name
        assert _rel(got, ref) <= 2e-2, (name, _rel(got, ref))
    # deterministic (no atomics)
    dq2, dk2, dv2 = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq2, dk=dk2, dv=dv2,
                         scratch=scr, impl=impl)
    torch.cuda.synchronize()
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)


@pytest.mark.parametrize("impl", [0, 1, 2], ids=["mma_sync", "tcgen05", "tcgen05_2tile"])
def test_attention_first_token_attends_only_to_itself(gpu_lib, impl):
    """Causal special case: row t = 0 of every sequence has o = v_0 exactly (up to
    the bf16 output rounding), lse = s_00, and dK/dV rows of the last key only
    receive gradient from the last query."""
    ee = gpu_lib
    B, T, Hq, Hkv = 2, 128, 2, 1
    n = B * T
    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    o = torch.empty_like(q)
    lse2 = torch.empty(n, Hq, device="cuda")
    ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl)
    torch.cuda.synchronize()
    for b in range(B):
        r = b * T
        for h in range(Hq):
            assert torch.equal(o[r, h * 128:(h + 1) * 128], v[r, :128])
            s00 = (q[r, h * 128:(h + 1) * 128].float() @ k[r, :128].float()) / math.sqrt(128)
            assert abs(lse2[r, h].item() * math.log(2.0) - s00.item()) <= 1e-3 * max(1, abs(s00))


@pytest.mark.parametrize("B,T,Hq,Hkv", [(2, 128, 4, 2), (1, 384, 2, 1), (3, 64, 8, 1),
                                        (1, 2048, 2, 2), (2, 192, 2, 1)])
def test_two_tile_forward_bitwise_equals_one_tile(gpu_lib, B, T, Hq, Hkv):
    """The ping-pong forward (two query tiles per CTA, impl 2) performs the same
    per-row operations in the same order as the one-tile kernel: o and lse2
    must be bitwise equal, including odd tile counts (T = 384, 192: the last
    CTA has one tile) and T = 64 (a single partial tile)."""
    ee = gpu_lib
    g = torch.Generator(device="cuda").manual_seed(T + Hq)
    n = B * T
    q = (torch.randn(n, Hq * 128, device="cuda", generator=g) * 3).bfloat16()
    k = (torch.randn(n, Hkv * 128, device="cuda", generator=g) * 3).bfloat16()
    v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
    outs = []
    for impl in (1, 2):
        o = torch.full_like(q, float("nan"))
        lse2 = torch.full((n, Hq), float("nan"), device="cuda")
        ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, impl=impl)
        torch.cuda.synchronize()
        outs.append((o, lse2))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
