"""The error floor of bf16 GEMM operands on the Layer exit's gain gradient
(A27): the fp64 oracle's own arithmetic, re-run with the CUDA path's
bf16 roundings (u1, q/k/v, P, o, u, [A|B], M, z, dS, dx1, [dA|dB], dO, the
attention dS, dq/dk/dv) and nothing else, already differs from the exact fp64
result by 1.5-3.0e-2 on g_att -- at or past the north_star bound -- while every other
tensor stays well inside it.  The two largest single contributors are the
FORWARD roundings of the QKV operand u1 and of q/k (peaked attention, score
std ~4, amplifies them), not anything the backward can repair.  This is why
tests/harness.py bounds g_att of Layer exits at 5e-2 (LAYER_GAIN_RTOL).
CPU only (no CUDA path involved)."""

import math

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from oracle import ee_oracle as O

ROUNDINGS = ("u1", "qkv", "P", "o", "u", "M", "AB", "z", "dS", "dx1", "dAB", "do", "dSa",
             "dqkv")


def _bf(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def layer_grads_emulated(p, x, y, at, R, alpha, eps=1e-5):
    """The oracle's Layer-exit forward/backward (oracle/ee_oracle.py) with bf16
    rounding applied at the points named in R.  Returns (g_att grad, W_q grad)."""
    T, Hq, Hkv = at["seq_len"], at["n_heads"], at["n_kv"]
    N, h = x.shape
    d = p["w_q"].shape[0] // Hq
    pos = np.arange(N) % T
    g = Hq // Hkv
    rr = lambda name, v: _bf(v) if name in R else v
    u1, r1, xh1 = O.rmsnorm(x, p["g_att"], eps)
    u1 = rr("u1", u1)
    q = rr("qkv", O.rope((u1 @ p["w_q"].T).reshape(N, Hq, d), pos, 1e4))
    k = rr("qkv", O.rope((u1 @ p["w_k"].T).reshape(N, Hkv, d), pos, 1e4))
    v = rr("qkv", (u1 @ p["w_v"].T).reshape(N, Hkv, d))
    P = O.attention_probs(q, k, T)
    o = np.zeros((N, Hq, d))
    for b in range(N // T):
        rs = slice(b * T, (b + 1) * T)
        for j in range(Hq):
            o[rs, j] = rr("P", P[b, j]) @ v[rs, j // g]
    o = rr("o", o.reshape(N, -1))
    x1 = x + o @ p["w_o"].T
    u, rx, xhat = O.rmsnorm(x1, p["g_a"], eps)
    u = rr("u", u)
    A = u @ p["w_gate"].T
    B = u @ p["w_up"].T
    M = rr("M", O.silu(A) * B)
    Ab, Bb = rr("AB", A), rr("AB", B)
    yv = x1 + M @ p["w_down"].T
    z, ry, yhat = O.rmsnorm(yv, p["g_f"], eps)
    z = rr("z", z)
    st = O.lm_loss_stats(z @ p["w_out"].T, y)
    W = st["valid"].sum()
    Pp = np.exp(z @ p["w_out"].T - st["lse"][:, None])
    oh = np.zeros_like(Pp)
    rows = np.nonzero(st["valid"])[0]
    oh[rows, y[rows]] = 1.0
    dS = rr("dS", (alpha * st["valid"] / W)[:, None] * (Pp - oh))
    dy, _ = O.rmsnorm_backward(dS @ p["w_out"], yhat, ry, p["g_f"])
    dM = rr("dx1", dy) @ p["w_down"]
    dA = rr("dAB", dM * Bb * O.silu_grad(Ab))
    dB = rr("dAB", dM * O.silu(Ab))
    dxn, _ = O.rmsnorm_backward(dA @ p["w_gate"] + dB @ p["w_up"], xhat, rx, p["g_a"])
    dx1 = rr("dx1", dy + dxn)
    do = rr("do", dx1 @ p["w_o"]).reshape(N, Hq, d)
    c = 1.0 / math.sqrt(d)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for b in range(N // T):
        rs = slice(b * T, (b + 1) * T)
        for j in range(Hq):
            Pj = P[b, j]
            dv[rs, j // g] += rr("P", Pj).T @ do[rs, j]
            dP = do[rs, j] @ v[rs, j // g].T
            dSa = rr("dSa", Pj * (dP - np.sum(dP * Pj, axis=1, keepdims=True)))
            dq[rs, j] = c * (dSa @ k[rs, j // g])
            dk[rs, j // g] += c * (dSa.T @ q[rs, j])
    dq = rr("dqkv", O.rope(dq, -pos, 1e4).reshape(N, -1))
    dk = rr("dqkv", O.rope(dk, -pos, 1e4).reshape(N, -1))
    dv = rr("dqkv", dv.reshape(N, -1))
    du1 = dq @ p["w_q"] + dk @ p["w_k"] + dv @ p["w_v"]
    return np.sum(du1 * xh1, axis=0), dq.T @ u1


def _inputs(seed):
    cfg = S.get_cfg("tiny_layer", seed=seed)
    cfg.tokens = 512
    p = {k: to_f64(v) for k, v in S.head_params(cfg)[1].items()}
    x = to_f64(S.hidden_states(cfg)[1])
    y = S.targets(cfg).numpy().astype(np.int64)
    return p, x, y, S.attn_geometry(cfg)


def test_emulation_without_roundings_is_the_oracle():
    p, x, y, at = _inputs(57)
    g, _ = layer_grads_emulated(p, x, y, at, set(), 0.5)
    ref = O.exit_loss_and_grads("layer", p, x, y, 0.5, 1e-5, attn=at).grads["g_att"]
    assert np.array_equal(g, ref) or np.linalg.norm(g - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("seed", [57, 63, 69])
def test_layer_gain_gradient_bf16_floor(seed):
    p, x, y, at = _inputs(seed)
    ref, ref_q = layer_grads_emulated(p, x, y, at, set(), 0.5)
    g, gq = layer_grads_emulated(p, x, y, at, set(ROUNDINGS), 0.5)
    e = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    eq = np.linalg.norm(gq - ref_q) / np.linalg.norm(ref_q)
    print(seed, f"g_att {e:.2e} w_q {eq:.2e}")
    assert 1.0e-2 <= e <= 4e-2            # at or past the north_star bound from bf16 operands alone
    assert eq <= 1.2e-2                   # the weight gradients keep their margin
    # the forward operand roundings of u1 and q/k dominate
    e_fwd = np.linalg.norm(layer_grads_emulated(p, x, y, at, {"u1", "qkv"}, 0.5)[0] - ref) \
        / np.linalg.norm(ref)
    assert e_fwd >= 0.5 * e
