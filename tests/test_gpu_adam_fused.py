"""Adam fused into the weight-gradient GEMM epilogues (include/ee.h
ee_tune_step_adam; ExitHeads.step_adam / step_host(lr=...)): bit-for-bit the
same parameters, moments, operands and losses as ee_tune_step followed by
ee_adam_update (forward, backward and update per exit), over several
steps, for every supported arch, ragged shapes and both weightings; and the
first update against the fp64 oracle's Adam (north_star tolerance)."""

import numpy as np
import pytest
import torch

import eesynth as S
from harness import GRAD_RTOL, rel_fro
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


def _heads(ee, cfg, params, n, weighting="uniform", grad_buffers=None):
    hd = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch,
                                  token_weighting=weighting), n, grad_buffers=grad_buffers)
    hd.init("copy", copy_src=[{k: v.cuda().float().contiguous() for k, v in p.items()}
                              for p in params], src_dtype=torch.float32)
    return hd


def _state(hd):
    return [{k: (hd.master[i][k].cpu(), hd.m[i][k].cpu(), hd.v[i][k].cpu(),
                 hd.operand[i][k].cpu()) for k in hd.master[i]} for i in range(hd.spec.num_exits)]


@pytest.mark.parametrize("arch,h,V,F,n,weighting", [
    ("embedding", 192, 2056, 0, 77, "uniform"),
    ("norm", 128, 1000, 0, 300, "uniform"),
    ("mlp", 128, 1000, 384, 300, "uniform"),
    ("mlp", 256, 4104, 512, 1000, "confidence"),
])
def test_fused_adam_bitwise_equals_step_then_adam(gpu_lib, arch, h, V, F, n, weighting):
    ee = gpu_lib
    cfg = S.Cfg(name="small", hidden=h, vocab=V, ffn=F, arch=arch, tokens=n, layers=2,
                after=[1, 2], init="random", seed=31)
    hidden = [x.cuda() for x in S.hidden_states(cfg, n, seed=4)]
    targets = S.targets(cfg, n, seed=4).cuda()
    params = S.head_params(cfg, seed=4)
    a = _heads(ee, cfg, params, n, weighting)
    b = _heads(ee, cfg, params, n, weighting)
    w = [1.0, 0.6]
    for it in range(3):
        lr = 1e-3 * (it + 1)
        la = a.step(hidden, targets, exit_weights=w).clone()
        a.adam(lr)
        lb = b.step_adam(hidden, targets, lr, exit_weights=w).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, lb), (it, la, lb)
    assert a.status() == (0, -1) and b.status() == (0, -1)
    sa, sb = _state(a), _state(b)
    for i in range(cfg.exits):
        for k in sa[i]:
            for j, nm in enumerate(("master", "m", "v", "operand")):
                assert torch.equal(sa[i][k][j], sb[i][k][j]), (i, k, nm)


def test_fused_adam_step_host_and_per_exit_buffers(gpu_lib):
    """The host-input API with lr (per-exit calls) equals step_adam on device
    inputs; shared gradient buffers (grad_buffers < E) do not matter to it."""
    ee = gpu_lib
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=256, layers=3,
                after=[1, 2, 3], init="random", seed=32)
    hidden = S.hidden_states(cfg, 256, seed=5)
    targets = S.targets(cfg, 256, seed=5)
    params = S.head_params(cfg, seed=5)
    a = _heads(ee, cfg, params, 256)
    b = _heads(ee, cfg, params, 256, grad_buffers=1)
    hh = [x.pin_memory() for x in hidden]
    th = targets.pin_memory()
    for it in range(2):
        a.step_adam([x.cuda() for x in hidden], targets.cuda(), 1e-3)
        b.step_host(hh, th, lr=1e-3)
    torch.cuda.synchronize()
    assert torch.equal(a.loss, b.loss)
    sa, sb = _state(a), _state(b)
    for i in range(cfg.exits):
        for k in sa[i]:
            for j in range(4):
                assert torch.equal(sa[i][k][j], sb[i][k][j]), (i, k, j)


def test_fused_adam_first_moment_matches_oracle_gradient(gpu_lib):
    """Step 1 from zero moments leaves m = (1 - beta1) g and v = (1 - beta2) g^2
    (A14): the gradients the fused epilogues consumed, read back from the
    moments, match the fp64 oracle's gradients (north_star tolerance, per
    tensor) -- the fused path never stores the gradient itself."""
    ee = gpu_lib
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300, layers=2,
                after=[1], init="random", seed=33)
    hidden = S.hidden_states(cfg, 300, seed=6)
    targets = S.targets(cfg, 300, seed=6)
    params = S.head_params(cfg, seed=6)
    hd = _heads(ee, cfg, params, 300)
    hd.step_adam([hidden[0].cuda()], targets.cuda(), 1e-3, beta1=0.9, beta2=0.95)
    torch.cuda.synchronize()
    from harness import oracle_exit
    res = oracle_exit("mlp", params[0], hidden[0], targets, 1.0)
    for k, g in res.grads.items():
        m = hd.m[0][k].cpu().double().numpy()
        v = hd.v[0][k].cpu().double().numpy()
        assert rel_fro(m / (1 - 0.9), g) <= GRAD_RTOL, k
        assert rel_fro(np.sqrt(v / (1 - 0.95)), np.abs(g)) <= GRAD_RTOL, k
        th, _, _ = O.adam_update(params[0][k].double().numpy(), m / (1 - 0.9), 0 * m, 0 * v,
                                 1e-3, 0.9, 0.95, 1e-5, 0.0, 1)
        got = hd.master[0][k].cpu().double().numpy()
        assert np.max(np.abs(got - th)) <= 1e-6 + 1e-6 * np.max(np.abs(th)), k


@pytest.mark.parametrize("grad_buffers", [None, 1, 2])
def test_adam_overlapped_on_side_stream_equals_sequential(gpu_lib, grad_buffers):
    """step_overlapped: exit i's Adam on a side stream overlapping exit i+1
    (and the next step), ordered by events -- bitwise the per-exit sequential
    update, also with shared gradient buffers."""
    ee = gpu_lib
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=256, layers=3,
                after=[1, 2, 3], init="random", seed=34)
    hidden = [x.cuda() for x in S.hidden_states(cfg, 256, seed=7)]
    targets = S.targets(cfg, 256, seed=7).cuda()
    params = S.head_params(cfg, seed=7)
    a = _heads(ee, cfg, params, 256)
    b = _heads(ee, cfg, params, 256, grad_buffers=grad_buffers)
    for it in range(3):
        lr = 1e-3 * (it + 1)
        a.step(hidden, targets)
        a.adam(lr)
        b.step_overlapped(hidden, targets, lr)
    b.join()
    torch.cuda.synchronize()
    assert torch.equal(a.loss, b.loss)
    sa, sb = _state(a), _state(b)
    for i in range(cfg.exits):
        for k in sa[i]:
            for j in range(4):
                assert torch.equal(sa[i][k][j], sb[i][k][j]), (i, k, j)


def test_fused_adam_layer_exit_bitwise(gpu_lib):
    """Layer exits (attention block + MLP): the attention weights' updates run
    after the GEMMs that read them (L7 before L6, L11 before L10); bitwise the
    separate step + Adam over two steps."""
    ee = gpu_lib
    cfg = S.get_cfg("tiny_layer", seed=35)
    hidden = [x.cuda() for x in S.hidden_states(cfg)]
    targets = S.targets(cfg).cuda()
    params = S.head_params(cfg)
    kw = dict(n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads, seq_len=cfg.seq_len)
    def mk():
        hd = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch, **kw),
                          cfg.tokens)
        hd.init("copy", copy_src=[{k: v.cuda().float().contiguous() for k, v in p.items()}
                                  for p in params], src_dtype=torch.float32)
        return hd
    a, b = mk(), mk()
    for it in range(2):
        a.step(hidden, targets)
        a.adam(1e-3 * (it + 1))
        b.step_adam(hidden, targets, 1e-3 * (it + 1))
    torch.cuda.synchronize()
    assert torch.equal(a.loss, b.loss)
    sa, sb = _state(a), _state(b)
    for i in range(cfg.exits):
        for k in sa[i]:
            for j in range(4):
                assert torch.equal(sa[i][k][j], sb[i][k][j]), (i, k, j)
