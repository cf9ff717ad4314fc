"""Pins for the fp64 oracle against what the paper and the mathematics fix.

Each test names the pin (P1..P14 in DESIGN.md §5) and the passage it follows.
None of these compares the oracle with itself: the references are hand-derived
worked examples (tests/golden), closed forms, invariants, library routines
(torch.nn.functional in fp64, scipy.special.logsumexp, torch.autograd) and
central finite differences.
"""

import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn
from scipy.special import logsumexp, softmax

from oracle import ee_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def _rng(seed):
    return np.random.default_rng(seed)


def _params(arch, h, V, F, rng, w_std=0.5):
    p = {"w_out": rng.normal(0, w_std, (V, h))}
    if arch != "embedding":
        p["g_f"] = 1.0 + 0.1 * rng.normal(size=h)
    if arch in ("mlp", "layer"):
        p["g_a"] = 1.0 + 0.1 * rng.normal(size=h)
        p["w_gate"] = rng.normal(0, w_std, (F, h))
        p["w_up"] = rng.normal(0, w_std, (F, h))
        p["w_down"] = rng.normal(0, w_std, (h, F))
    if arch == "layer":   # 2 query heads sharing 1 kv head (GQA), d = h / 2
        p["g_att"] = 1.0 + 0.1 * rng.normal(size=h)
        p["w_q"] = rng.normal(0, w_std, (h, h))
        p["w_k"] = rng.normal(0, w_std, (h // 2, h))
        p["w_v"] = rng.normal(0, w_std, (h // 2, h))
        p["w_o"] = rng.normal(0, w_std, (h, h))
    return p


def _attn(arch, N, T=None):
    """Attention geometry of the test Layer exits: 2 heads, 1 kv head, and
    sequences of T tokens (default: two sequences when N is even)."""
    if arch != "layer":
        return None
    T = T or (N // 2 if N % 2 == 0 else N)
    return {"seq_len": T, "n_heads": 2, "n_kv": 1, "theta": 10000.0}


def _elg(arch, p, x, y, alpha, eps, **kw):
    return O.exit_loss_and_grads(arch, p, x, y, alpha, eps, attn=_attn(arch, x.shape[0]), **kw)


# --------------------------------------------------------------------------- P1, P2
def test_P1_worked_example_embedding():
    g = json.load(open(GOLDEN))["P1_embedding"]
    p = {"w_out": np.array(g["w_out"])}
    r = O.exit_loss_and_grads("embedding", p, np.array(g["z"]), np.array(g["target"]), 1.0, 0.0,
                              keep_act=True)
    assert r.stats["lse"][0] == pytest.approx(g["lse"], rel=1e-14)
    assert r.loss == pytest.approx(g["loss"], rel=1e-13)
    assert r.stats["conf"][0] == pytest.approx(g["conf"], rel=1e-13)
    assert r.stats["argmax"][0] == g["argmax"]
    np.testing.assert_allclose(r.grads["w_out"], np.array(g["dW_out"]), rtol=1e-13)
    # dz is not a parameter gradient of an Embedding exit; check it via the Norm path
    # identity dz = dS W_out using the golden dS.
    np.testing.assert_allclose(np.array(g["dS"]) @ p["w_out"], np.array(g["dz"]), rtol=1e-12)


def test_P2_worked_example_norm_and_scale_invariance():
    g = json.load(open(GOLDEN))["P2_norm"]
    p = {"w_out": np.array(g["w_out"]), "g_f": np.array(g["g_f"])}
    x = np.array(g["x"])
    r = O.exit_loss_and_grads("norm", p, x, np.array(g["target"]), 1.0, g["eps"], keep_act=True)
    assert r.act["r_y"][0] == pytest.approx(g["r"], rel=1e-14)
    np.testing.assert_allclose(r.act["yhat"][0], g["yhat"], rtol=1e-14)
    assert r.stats["lse"][0] == pytest.approx(g["lse"], rel=1e-14)
    assert r.loss == pytest.approx(g["loss"], rel=1e-13)
    np.testing.assert_allclose(r.grads["g_f"], g["dg_f"], rtol=1e-12)
    # P5: at eps = 0 RMSNorm is scale invariant, so x . dx = 0 for any cotangent.
    dz = np.array([[0.3, -1.7]])
    dx, _ = O.rmsnorm_backward(dz, r.act["yhat"], r.act["r_y"], p["g_f"])
    assert abs(float(np.sum(x * dx))) < 1e-14


# --------------------------------------------------------------------------- P3
@pytest.mark.parametrize("arch", O.ARCHS)
def test_P3_uniform_logits_closed_form(arch):
    rng = _rng(3)
    h, V, F, N = 8, 512, 12, 16
    p = _params(arch, h, V, F, rng)
    p["w_out"][:] = 0.0
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    y[3] = -1
    alpha = 0.7
    r = _elg(arch, p, x, y, alpha, 1e-5, keep_act=True)
    assert r.loss == pytest.approx(math.log(512), rel=1e-15)       # ln V
    assert math.log(512) == pytest.approx(6.238324625039508, rel=1e-15)
    np.testing.assert_allclose(r.stats["conf"], 1.0 / V, rtol=1e-14)
    # dW_out[v] = alpha/W sum_t w_t (1/V - 1[y_t = v]) z_t
    w = (y != -1).astype(float)
    W = w.sum()
    onehot = np.zeros((N, V))
    onehot[np.nonzero(w)[0], y[w > 0]] = 1
    expect = alpha / W * ((w[:, None] * (1.0 / V - onehot)).T @ r.act["z"])
    np.testing.assert_allclose(r.grads["w_out"], expect, rtol=1e-12, atol=1e-15)
    # dz = dS W_out = 0 exactly, so every gradient below W_out is exactly zero.
    for k in ("g_f", "g_a", "w_gate", "w_up", "w_down", "g_att", "w_q", "w_k", "w_v", "w_o"):
        if k in r.grads:
            assert np.all(r.grads[k] == 0.0), k


def test_P3_uniform_logits_vocab_32000():
    p = {"w_out": np.zeros((32000, 8))}
    x = _rng(0).normal(size=(3, 8))
    r = O.exit_loss_and_grads("embedding", p, x, np.array([0, 31999, 5]), 1.0, 0.0)
    assert r.loss == pytest.approx(10.373491181781864, rel=1e-15)   # ln 32000


# --------------------------------------------------------------------------- P4
@pytest.mark.parametrize("arch", O.ARCHS)
def test_P4_softmax_ce_gradient_rows_sum_to_zero(arch):
    rng = _rng(4)
    h, V, F, N = 16, 40, 24, 32
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    r = _elg(arch, p, x, y, 1.3, 1e-5)
    col = r.grads["w_out"].sum(axis=0)
    assert np.max(np.abs(col)) <= 1e-13 * np.max(np.abs(r.grads["w_out"])) * V


# --------------------------------------------------------------------------- P5
def test_P5_rmsnorm_scale_invariance_and_textbook():
    rng = _rng(5)
    x = rng.normal(size=(7, 33))
    g = 1 + 0.1 * rng.normal(size=33)
    a, _, _ = O.rmsnorm(x, g, 0.0)
    b, _, _ = O.rmsnorm(3.7 * x, g, 0.0)
    np.testing.assert_allclose(a, b, rtol=1e-14)
    # library routine: torch.nn.functional.rms_norm in fp64
    ref = Fn.rms_norm(torch.from_numpy(x), (33,), torch.from_numpy(g), eps=1e-5).numpy()
    np.testing.assert_allclose(O.rmsnorm(x, g, 1e-5)[0], ref, rtol=1e-13)


# --------------------------------------------------------------------------- P6
@pytest.mark.parametrize("arch", O.ARCHS)
def test_P6_central_finite_differences(arch):
    """Every parameter tensor of every architecture; fp64, step 1e-6."""
    rng = _rng(6)
    h, V, F, N = 8, 16, 12, 4
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = np.array([3, -1, 15, 0])
    alpha, eps = 0.8, 1e-5
    r = _elg(arch, p, x, y, alpha, eps)

    def f(pp):
        return alpha * _elg(arch, pp, x, y, alpha, eps).loss

    step = 1e-6
    for name, val in p.items():
        num = np.zeros_like(val)
        it = np.nditer(val, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            q = {k: v.copy() for k, v in p.items()}
            q[name][idx] += step
            fp = f(q)
            q[name][idx] -= 2 * step
            fm = f(q)
            num[idx] = (fp - fm) / (2 * step)
        err = np.linalg.norm(num - r.grads[name]) / max(np.linalg.norm(r.grads[name]), 1e-30)
        assert err <= 1e-6, (arch, name, err)


# --------------------------------------------------------------------------- P7
def test_P7_copy_init_reproduces_original_head_bitwise():
    """A Norm exit at the last layer, copy-initialised, gives exactly the
    original model's logits and loss."""
    rng = _rng(7)
    h, V, N = 64, 512, 32
    bb = {"final_norm": 1 + 0.1 * rng.normal(size=h), "w_out": rng.normal(0, h ** -0.5, (V, h)),
          "layers": []}
    h_last = rng.normal(size=(N, h))
    p = O.init_copy("norm", bb, after_layer=2)
    assert np.array_equal(p["w_out"], bb["w_out"]) and np.array_equal(p["g_f"], bb["final_norm"])
    assert not np.shares_memory(p["w_out"], bb["w_out"])               # deep copy
    S_exit = O.exit_forward("norm", p, h_last, 1e-5)["S"]
    S_orig = O.original_final_logits(bb, h_last, 1e-5)
    assert np.array_equal(S_exit, S_orig)
    y = rng.integers(0, V, N)
    l_exit = O.lm_loss_stats(S_exit, y)["loss"].mean()
    l_orig = np.mean(logsumexp(S_orig, axis=1) - S_orig[np.arange(N), y])
    assert l_exit == pytest.approx(l_orig, rel=1e-14)
    p["w_out"][0, 0] += 1.0                                           # mutate exit ...
    assert p["w_out"][0, 0] != bb["w_out"][0, 0]                      # ... source untouched


def test_P7_copy_init_mlp_structure():
    rng = _rng(8)
    h, V, F = 8, 16, 12
    layers = [{"mlp_norm": rng.normal(size=h), "w_gate": rng.normal(size=(F, h)),
               "w_up": rng.normal(size=(F, h)), "w_down": rng.normal(size=(h, F))} for _ in range(3)]
    bb = {"final_norm": rng.normal(size=h), "w_out": rng.normal(size=(V, h)), "layers": layers}
    p = O.init_copy("mlp", bb, after_layer=2)
    assert np.array_equal(p["w_gate"], layers[1]["w_gate"])
    assert np.array_equal(p["g_a"], layers[1]["mlp_norm"])
    assert np.array_equal(p["w_down"], layers[1]["w_down"])
    pe = O.init_copy("embedding", bb, after_layer=2)
    assert set(pe) == {"w_out"}
    with pytest.raises(LookupError):
        O.init_copy("mlp", bb, after_layer=4)
    with pytest.raises(LookupError):
        O.init_copy("norm", {"w_out": bb["w_out"], "final_norm": None}, after_layer=1)


# --------------------------------------------------------------------------- P8, P9
def test_P8_two_class_softplus():
    rng = _rng(9)
    S = rng.normal(size=(10, 2)) * 3
    y = rng.integers(0, 2, 10)
    st = O.lm_loss_stats(S, y)
    other = S[np.arange(10), 1 - y]
    np.testing.assert_allclose(st["loss"], np.logaddexp(0.0, other - S[np.arange(10), y]), rtol=1e-10,
                               atol=1e-15)


@pytest.mark.parametrize("arch", O.ARCHS)
def test_P8_P9_against_torch_library_and_autograd(arch):
    """Forward via torch.nn.functional library routines (rms_norm, silu,
    linear, cross_entropy with ignore_index) in fp64; gradients via autograd."""
    rng = _rng(10)
    h, V, F, N = 24, 50, 40, 30
    p = _params(arch, h, V, F, rng, w_std=0.3)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    y[[2, 11]] = -1
    alpha, eps = 1.7, 1e-5
    r = _elg(arch, p, x, y, alpha, eps, keep_act=True)

    tp = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    tx = torch.tensor(x)
    t = tx
    if arch == "layer":  # F.scaled_dot_product_attention (causal, GQA); RoPE rotate-half
        T, d = N // 2, h // 2
        u = Fn.rms_norm(tx, (h,), tp["g_att"], eps)
        pos = torch.arange(N) % T
        inv = 10000.0 ** (-torch.arange(d // 2, dtype=torch.float64) * 2 / d)
        ang = pos[:, None].double() * inv[None]

        def rot(zz):
            z1, z2 = zz[..., :d // 2], zz[..., d // 2:]
            c, s_ = torch.cos(ang)[:, None], torch.sin(ang)[:, None]
            return torch.cat([z1 * c - z2 * s_, z2 * c + z1 * s_], -1)
        q = rot(Fn.linear(u, tp["w_q"]).view(N, 2, d)).view(2, T, 2, d).transpose(1, 2)
        k = rot(Fn.linear(u, tp["w_k"]).view(N, 1, d)).view(2, T, 1, d).transpose(1, 2)
        v = Fn.linear(u, tp["w_v"]).view(2, T, 1, d).transpose(1, 2)
        o = Fn.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        tx = tx + Fn.linear(o.transpose(1, 2).reshape(N, h), tp["w_o"])
        t = tx
    if arch in ("mlp", "layer"):
        u = Fn.rms_norm(tx, (h,), tp["g_a"], eps)
        m = Fn.silu(Fn.linear(u, tp["w_gate"])) * Fn.linear(u, tp["w_up"])
        t = tx + Fn.linear(m, tp["w_down"])
    if arch != "embedding":
        t = Fn.rms_norm(t, (h,), tp["g_f"], eps)
    logits = Fn.linear(t, tp["w_out"])
    loss = Fn.cross_entropy(logits, torch.tensor(y, dtype=torch.long), ignore_index=-1)
    (alpha * loss).backward()
    assert r.loss == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(r.stats["lse"], logsumexp(r.act["S"], axis=1), rtol=1e-13)
    np.testing.assert_allclose(r.stats["conf"], softmax(r.act["S"], axis=1).max(axis=1), rtol=1e-12)
    for k in p:
        np.testing.assert_allclose(r.grads[k], tp[k].grad.numpy(), rtol=1e-10, atol=1e-14,
                                   err_msg=f"{arch}:{k}")


# --------------------------------------------------------------------------- P10, P11
@pytest.mark.parametrize("arch", ("norm", "mlp"))
def test_P10_data_parallel_sharding_linearity(arch):
    """With the global valid count W, gradients over token shards sum to the
    full-batch gradient and losses sum to the full mean (A16)."""
    rng = _rng(11)
    h, V, F, N = 12, 30, 20, 40
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    y[[0, 7, 33]] = -1
    full = O.exit_loss_and_grads(arch, p, x, y, 0.9, 1e-5)
    W = int(np.sum(y != -1))
    shards = [O.exit_loss_and_grads(arch, p, x[s], y[s], 0.9, 1e-5, valid_count=W)
              for s in (slice(0, 13), slice(13, 29), slice(29, 40))]
    assert sum(s.loss for s in shards) == pytest.approx(full.loss, rel=1e-13)
    for k in p:
        np.testing.assert_allclose(sum(s.grads[k] for s in shards), full.grads[k], rtol=1e-11,
                                   atol=1e-15)


def test_P11_exit_independence():
    rng = _rng(12)
    h, V, F, N = 8, 20, 10, 12
    pa, pb = _params("mlp", h, V, F, rng), _params("mlp", h, V, F, rng)
    xa, xb = rng.normal(size=(N, h)), rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    la, ga, _ = O.tune_step("mlp", [pa], [xa], y, [1.0], 1e-5)
    lab, gab, _ = O.tune_step("mlp", [pa, pb], [xa, xb], y, [1.0, 0.5], 1e-5)
    assert la[0] == lab[0]
    for k in pa:
        assert np.array_equal(ga[0][k], gab[0][k])


# --------------------------------------------------------------------------- P12, P13
def test_P12_degenerate_weights():
    rng = _rng(13)
    h, V, F, N = 8, 20, 10, 12
    p = _params("mlp", h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    r = O.exit_loss_and_grads("mlp", p, x, y, 0.0, 1e-5)               # alpha = 0
    assert r.loss > 0
    for k, g in r.grads.items():
        assert np.all(g == 0.0), k
    m = np.zeros_like(p["w_out"])
    th, _, _ = O.adam_update(p["w_out"], r.grads["w_out"], m, m.copy(), 1e-4, 0.9, 0.95, 1e-5, 0.0, 1)
    assert np.array_equal(th, p["w_out"])                              # params bitwise unchanged
    r2 = O.exit_loss_and_grads("mlp", p, x, np.full(N, -1), 1.0, 1e-5)  # all ignored
    assert r2.loss == 0.0
    for g in r2.grads.values():
        assert np.all(g == 0.0)


def test_P13_adam_first_step_closed_form():
    rng = _rng(14)
    th = rng.normal(size=1000)
    g = rng.normal(size=1000) * 10 ** rng.uniform(-6, 1, 1000)
    lr, eps = 1e-4, 1e-5
    new, m, v = O.adam_update(th, g, np.zeros(1000), np.zeros(1000), lr, 0.9, 0.95, eps, 0.0, 1)
    np.testing.assert_allclose(new, th - lr * g / (np.abs(g) + eps), rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(m, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v, 0.05 * g * g, rtol=1e-14)
    # weight decay adds -lr*wd*theta
    new2, _, _ = O.adam_update(th, g, np.zeros(1000), np.zeros(1000), lr, 0.9, 0.95, eps, 0.01, 1)
    np.testing.assert_allclose(new2 - new, -lr * 0.01 * th, rtol=1e-9, atol=1e-20)
    # SGD
    s, _ = O.sgd_update(th, g, None, 0.5, 0.0)
    np.testing.assert_allclose(s, th - 0.5 * g, rtol=1e-15)


@pytest.mark.parametrize("wd", [0.0, 0.01])
@pytest.mark.parametrize("grad_scale", [1.0, 0.25])
def test_P13_adam_multi_step_against_torch_optim(wd, grad_scale):
    """P:374-375 (Adam, beta1 0.9, beta2 0.95, eps 1e-5) over 6 steps with fresh
    random gradients each step, against torch.optim.AdamW in fp64 (decoupled
    weight decay; = torch.optim.Adam at wd 0).  Pins the moment decays and the
    bias corrections at t > 1, which the t = 1 closed form cannot see (a
    beta1/beta2 swap in v passes P13 and fails here)."""
    rng = _rng(140)
    th0 = rng.normal(size=(7, 33))
    lrs = [1e-3, 5e-4, 2e-3, 1e-4, 7e-4, 3e-4]
    t = torch.tensor(th0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([t], lr=lrs[0], betas=(0.9, 0.95), eps=1e-5, weight_decay=wd)
    th, m, v = th0.copy(), np.zeros_like(th0), np.zeros_like(th0)
    for step, lr in enumerate(lrs, start=1):
        g = rng.normal(size=th0.shape) * 10 ** rng.uniform(-4, 1, th0.shape)
        th, m, v = O.adam_update(th, g, m, v, lr, 0.9, 0.95, 1e-5, wd, step, grad_scale)
        for grp in opt.param_groups:
            grp["lr"] = lr
        t.grad = torch.tensor(g * grad_scale)
        opt.step()
        np.testing.assert_allclose(th, t.detach().numpy(), rtol=1e-12, atol=1e-15)
        st = opt.state[t]
        np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-13, atol=0)
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-13, atol=0)


@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_P13_sgd_momentum_against_torch_optim(momentum):
    """SGD (the ee_sgd_update alternative) with heavy-ball momentum b = mu b + g
    (b_1 = g), theta -= lr b, over 5 steps against torch.optim.SGD in fp64."""
    rng = _rng(141)
    th0 = rng.normal(size=(5, 17))
    t = torch.tensor(th0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([t], lr=0.1, momentum=momentum)
    th, buf = th0.copy(), None
    for _ in range(5):
        g = rng.normal(size=th0.shape)
        th, buf = O.sgd_update(th, g, buf, 0.1, momentum, grad_scale=0.5)
        t.grad = torch.tensor(0.5 * g)
        opt.step()
        np.testing.assert_allclose(th, t.detach().numpy(), rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------------------- P14
def test_P14_lr_schedule_and_token_budget():
    T = 40000
    w = math.ceil(0.01 * T)
    assert O.lr_at(w, T) == pytest.approx(1e-4, rel=1e-15)             # "maximum ... 10^-4"
    assert O.lr_at(T, T) == pytest.approx(1e-5, rel=1e-15)             # "minimum of 10^-5"
    assert O.lr_at(0, T) == 0.0
    assert O.lr_at(w // 2, T) == pytest.approx(0.5e-4, rel=1e-15)
    assert O.lr_at((w + T) // 2, T) == pytest.approx(0.55e-4, rel=1e-12)
    with pytest.raises(ValueError):
        O.lr_at(T + 1, T)
    assert O.token_budget() == 1_310_720_000


# --------------------------------------------------------------------------- A6, A9
def test_targets_out_of_range_and_argmax_ties():
    S = np.array([[1.0, 3.0, 3.0, 0.0], [2.0, 2.0, 2.0, 2.0]])
    st = O.lm_loss_stats(S, np.array([1, -1]))
    assert list(st["argmax"]) == [1, 0]                                # lowest index on ties
    assert st["loss"][1] == 0.0
    with pytest.raises(ValueError):
        O.lm_loss_stats(S, np.array([4, 0]))
    with pytest.raises(ValueError):
        O.lm_loss_stats(S, np.array([-2, 0]))


def test_bf16_widening_is_exact():
    t = torch.randn(1000).to(torch.bfloat16)
    bits = t.view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(O.bf16_bits_to_f64(bits), t.to(torch.float64).numpy())


# --------------------------------------------------------------------------- A17 (NEXT #1)
@pytest.mark.parametrize("arch", O.ARCHS)
def test_confidence_weighting_detached_and_identity(arch):
    """Dynamic token-wise weights: w_t = c_t = max
    softmax prob, detached.  Pins: (i) explicit all-ones weights reproduce the
    static loss and gradients bitwise; (ii) c_t is the max softmax probability
    (scipy); (iii) the gradient equals central finite differences of
    sum_t c_t loss_t(theta) / sum_t c_t with c held at its value at theta_0."""
    rng = _rng(21)
    h, V, F, N = 8, 16, 12, 6
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = np.array([3, -1, 15, 0, 7, 7])
    alpha, eps = 0.9, 1e-5
    r_u = _elg(arch, p, x, y, alpha, eps)
    r_1 = _elg(arch, p, x, y, alpha, eps, weighting=np.ones(N))
    assert r_1.loss == r_u.loss
    for k in p:
        assert np.array_equal(r_1.grads[k], r_u.grads[k]), k
    r_c = _elg(arch, p, x, y, alpha, eps, keep_act=True, weighting="confidence")
    c = softmax(r_c.act["S"], axis=1).max(axis=1)
    np.testing.assert_allclose(r_c.stats["conf"], c, rtol=1e-13)
    valid = y != -1
    L_expect = np.sum(c[valid] * r_c.stats["loss"][valid]) / np.sum(c[valid])
    assert r_c.loss == pytest.approx(L_expect, rel=1e-13)

    def f(pp):  # c held fixed (detached)
        return alpha * _elg(arch, pp, x, y, alpha, eps, weighting=c).loss

    step = 1e-6
    for name, val in p.items():
        num = np.zeros_like(val)
        it = np.nditer(val, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            q = {k: v.copy() for k, v in p.items()}
            q[name][idx] += step
            fp = f(q)
            q[name][idx] -= 2 * step
            num[idx] = (fp - f(q)) / (2 * step)
        err = np.linalg.norm(num - r_c.grads[name]) / max(np.linalg.norm(r_c.grads[name]), 1e-30)
        assert err <= 1e-6, (arch, name, err)


def test_confidence_weighting_uniform_logits():
    """W_out = 0: every c_t = 1/V, so confidence weighting = uniform: loss ln V."""
    p = {"w_out": np.zeros((64, 8))}
    x = _rng(0).normal(size=(5, 8))
    r = O.exit_loss_and_grads("embedding", p, x, np.array([0, 1, 2, -1, 63]), 1.0, 0.0,
                              weighting="confidence")
    assert r.loss == pytest.approx(math.log(64), rel=1e-14)


def test_exit_infer_thresholds():
    """Confidence-based early exit: threshold 1 disables exits
    (P:385); threshold 0 exits every token at the first exit; with W_out = 0 the
    confidence is exactly 1/V (uniform)."""
    rng = _rng(30)
    h, V, F, N = 8, 20, 12, 9
    ps = [_params("mlp", h, V, F, rng) for _ in range(3)]
    xs = [rng.normal(size=(N, h)) for _ in range(3)]
    am, cf, first = O.exit_infer("mlp", ps, xs, 1.0, 1e-5)
    assert np.all(first == -1) and np.all(cf < 1.0)
    _, _, first0 = O.exit_infer("mlp", ps, xs, 0.0, 1e-5)
    assert np.all(first0 == 0)
    tau = float(np.median(cf[1]))
    _, _, f = O.exit_infer("mlp", ps, xs, tau, 1e-5)
    for t in range(N):
        expect = next((i for i in range(3) if cf[i, t] >= tau), -1)
        assert f[t] == expect
    p0 = dict(ps[0], w_out=np.zeros((V, h)))
    _, c0, _ = O.exit_infer("mlp", [p0], [xs[0]], 0.5, 1e-5)
    np.testing.assert_allclose(c0, 1.0 / V, rtol=1e-14)
    for i in range(3):
        S = O.exit_forward("mlp", ps[i], xs[i], 1e-5)["S"]
        np.testing.assert_array_equal(am[i], np.argmax(S, axis=1))


# --------------------------------------------------------------------------- NEXT #3
def _layer(rng, h, nh, nkv, F, std=0.3):
    d = h // nh
    return {"g_att": 1 + 0.1 * rng.normal(size=h), "w_q": rng.normal(0, std, (nh * d, h)),
            "w_k": rng.normal(0, std, (nkv * d, h)), "w_v": rng.normal(0, std, (nkv * d, h)),
            "w_o": rng.normal(0, std, (h, nh * d)), "g_mlp": 1 + 0.1 * rng.normal(size=h),
            "w_gate": rng.normal(0, std, (F, h)), "w_up": rng.normal(0, std, (F, h)),
            "w_down": rng.normal(0, std, (h, F))}


def test_rope_is_a_relative_rotation():
    """RoPE preserves norms and q_m . k_n depends only on m - n."""
    rng = _rng(40)
    d = 16
    q = rng.normal(size=(1, 1, d))
    k = rng.normal(size=(1, 1, d))
    for m in (0, 3, 100):
        np.testing.assert_allclose(np.linalg.norm(O.rope(q, np.array([m]))), np.linalg.norm(q),
                                   rtol=1e-13)
    dot = lambda m, n: float(np.sum(O.rope(q, np.array([m])) * O.rope(k, np.array([n]))))
    assert dot(7, 3) == pytest.approx(dot(104, 100), rel=1e-11)
    assert dot(0, 0) == pytest.approx(float(np.sum(q * k)), rel=1e-13)


@pytest.mark.parametrize("nh,nkv", [(4, 4), (4, 2)])
def test_llama_layer_matches_torch_sdpa(nh, nkv):
    """One layer vs a composition of torch library routines in fp64:
    F.rms_norm, F.scaled_dot_product_attention(is_causal, GQA), F.silu; RoPE
    written out (rotate-half) and pinned separately above."""
    rng = _rng(41)
    h, F, T, B = 32, 24, 6, 2
    L = _layer(rng, h, nh, nkv, F)
    x = rng.normal(size=(B * T, h))
    got = O.llama_layer_forward(L, x, T, nh, nkv, 1e-5)
    t = {k: torch.tensor(v) for k, v in L.items()}
    X = torch.tensor(x)
    d = h // nh
    u = Fn.rms_norm(X, (h,), t["g_att"], 1e-5)
    pos = torch.arange(B * T) % T
    inv = 10000.0 ** (-torch.arange(d // 2, dtype=torch.float64) * 2 / d)
    ang = pos[:, None].double() * inv[None]

    def rot(z):
        z1, z2 = z[..., :d // 2], z[..., d // 2:]
        c, s = torch.cos(ang)[:, None], torch.sin(ang)[:, None]
        return torch.cat([z1 * c - z2 * s, z2 * c + z1 * s], -1)
    q = rot(Fn.linear(u, t["w_q"]).view(B * T, nh, d)).view(B, T, nh, d).transpose(1, 2)
    k = rot(Fn.linear(u, t["w_k"]).view(B * T, nkv, d)).view(B, T, nkv, d).transpose(1, 2)
    v = Fn.linear(u, t["w_v"]).view(B, T, nkv, d).transpose(1, 2)
    o = Fn.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=nkv != nh)
    X = X + Fn.linear(o.transpose(1, 2).reshape(B * T, nh * d), t["w_o"])
    u2 = Fn.rms_norm(X, (h,), t["g_mlp"], 1e-5)
    X = X + Fn.linear(Fn.silu(Fn.linear(u2, t["w_gate"])) * Fn.linear(u2, t["w_up"]), t["w_down"])
    np.testing.assert_allclose(got, X.numpy(), rtol=1e-11, atol=1e-12)


def test_backbone_partial_forward_structure():
    """Zero output projections make a layer the identity (pure residual);
    the partial forward stops at the last exit layer and returns the
    states after the requested layers; sequences do not attend across each
    other (causal within each seq_len block)."""
    rng = _rng(42)
    h, nh, nkv, F, T = 16, 2, 1, 12, 5
    layers = [_layer(rng, h, nh, nkv, F) for _ in range(4)]
    x0 = rng.normal(size=(2 * T, h))
    z = dict(layers[0], w_o=np.zeros((h, h)), w_down=np.zeros((h, F)))
    np.testing.assert_array_equal(O.llama_layer_forward(z, x0, T, nh, nkv, 1e-5), x0)
    outs = O.backbone_forward(layers, x0, T, nh, nkv, [1, 3], 1e-5)
    x1 = O.llama_layer_forward(layers[0], x0, T, nh, nkv, 1e-5)
    x3 = O.llama_layer_forward(layers[2], O.llama_layer_forward(layers[1], x1, T, nh, nkv, 1e-5),
                               T, nh, nkv, 1e-5)
    np.testing.assert_array_equal(outs[0], x1)
    np.testing.assert_array_equal(outs[1], x3)
    x_mod = x0.copy()
    x_mod[T:] += 1.0                                                  # change sequence 2 only
    np.testing.assert_array_equal(O.llama_layer_forward(layers[0], x_mod, T, nh, nkv, 1e-5)[:T], x1[:T])
    x_fut = x0.copy()
    x_fut[T - 1] += 1.0                                               # change the last token
    np.testing.assert_array_equal(O.llama_layer_forward(layers[0], x_fut, T, nh, nkv, 1e-5)[:T - 1],
                                  x1[:T - 1])


# --------------------------------------------------------------------------- NEXT #2: Layer exit
def test_P10_layer_data_parallel_over_whole_sequences():
    """Layer exits couple tokens within a sequence, so DP shards are whole
    sequences; with the global W the shard gradients sum to the full batch's."""
    rng = _rng(50)
    h, V, F, T = 8, 30, 12, 5
    N = 4 * T
    p = _params("layer", h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    y[[0, 7, 13]] = -1
    at = _attn("layer", N, T)
    full = O.exit_loss_and_grads("layer", p, x, y, 0.9, 1e-5, attn=at)
    W = int(np.sum(y != -1))
    shards = [O.exit_loss_and_grads("layer", p, x[s], y[s], 0.9, 1e-5, valid_count=W, attn=at)
              for s in (slice(0, T), slice(T, 3 * T), slice(3 * T, N))]
    assert sum(s.loss for s in shards) == pytest.approx(full.loss, rel=1e-13)
    for k in p:
        np.testing.assert_allclose(sum(s.grads[k] for s in shards), full.grads[k], rtol=1e-10,
                                   atol=1e-14, err_msg=k)


def test_layer_exit_uniform_attention_closed_form():
    """W_q = W_k = 0: every score is 0, so token t attends uniformly to the
    t+1 positions s <= t of its own sequence: x1_t = x_t + W_o (mean_{s<=t} v_s)
    per query head (GQA: both heads read kv head 0)."""
    rng = _rng(51)
    h, V, F, T = 8, 16, 12, 6
    N = 2 * T
    p = _params("layer", h, V, F, rng)
    p["w_q"][:] = 0.0
    p["w_k"][:] = 0.0
    x = rng.normal(size=(N, h))
    act = O.exit_forward("layer", p, x, 1e-5, _attn("layer", N, T))
    u1 = O.rmsnorm(x, p["g_att"], 1e-5)[0]
    v = u1 @ p["w_v"].T                                              # [N, d], one kv head
    o = np.zeros((N, h))
    for b in range(2):
        for t in range(T):
            m = v[b * T:b * T + t + 1].mean(axis=0)
            o[b * T + t] = np.concatenate([m, m])                    # both query heads
    np.testing.assert_allclose(act["x1"], x + o @ p["w_o"].T, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(act["x1"][0], x[0] + np.concatenate([v[0], v[0]]) @ p["w_o"].T,
                               rtol=1e-13)                           # t = 0 sees only itself


def test_layer_exit_copy_of_last_layer_skips_one_layer():
    """P:237 + P:242: a Layer exit after layer L-1, initialised as a copy of the
    last layer L (plus final norm and W_out), reproduces the original model's
    output on the same input: the exit *is* layer L followed by the final head.
    Cross-checks the exit's forward against llama_layer_forward (independent
    code, pinned to torch SDPA above)."""
    rng = _rng(52)
    h, nh, nkv, F, T, V, Lyr = 16, 2, 1, 12, 5, 40, 3
    layers = [_layer(rng, h, nh, nkv, F) for _ in range(Lyr)]
    for L in layers:
        L["mlp_norm"] = L["g_mlp"]
    bb = {"final_norm": 1 + 0.1 * rng.normal(size=h), "w_out": rng.normal(0, 0.3, (V, h)),
          "layers": layers}
    x0 = rng.normal(size=(2 * T, h))
    h_prev, h_last = O.backbone_forward(layers, x0, T, nh, nkv, [Lyr - 1, Lyr], 1e-5)
    p = O.init_copy("layer", bb, after_layer=Lyr - 1)
    assert np.array_equal(p["w_q"], layers[-1]["w_q"]) and not np.shares_memory(p["w_q"], layers[-1]["w_q"])
    assert np.array_equal(p["g_a"], layers[-1]["g_mlp"])
    at = {"seq_len": T, "n_heads": nh, "n_kv": nkv, "theta": 10000.0}
    S_exit = O.exit_forward("layer", p, h_prev, 1e-5, at)["S"]
    S_orig = O.original_final_logits(bb, h_last, 1e-5)
    np.testing.assert_allclose(S_exit, S_orig, rtol=1e-12, atol=1e-12)
    # copying is position-independent (always the LAST layer)
    p1 = O.init_copy("layer", bb, after_layer=1)
    assert all(np.array_equal(p1[k], p[k]) for k in p)
    with pytest.raises(LookupError):
        O.init_copy("layer", dict(bb, layers=[{k: v for k, v in layers[0].items() if k != "w_o"}]), 1)
    with pytest.raises(ValueError):                                  # tokens not whole sequences
        O.exit_forward("layer", p, h_prev[:7], 1e-5, at)
