"""Initialisers (Copy / Random) and optimizers (Adam P:374-375, SGD)
on the GPU, against the oracle and the statistical pins (P7, P12, P13, P15)."""

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from harness import gpu_step, oracle_exit
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


def _store(ee, cfg, n=0):
    spec = ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch)
    return ee.ExitHeads(spec, max_tokens=max(n, 1))


def _copy_src(cfg, bb):
    src = []
    for k in cfg.after:
        d = {"w_out": bb["w_out"].cuda()}
        if cfg.arch in ("norm", "mlp"):
            d["g_f"] = bb["final_norm"].cuda()
        if cfg.arch == "mlp":
            L = bb["layers"][k]
            d.update(g_a=L["mlp_norm"].cuda(), w_gate=L["w_gate"].cuda(), w_up=L["w_up"].cuda(),
                     w_down=L["w_down"].cuda())
        src.append(d)
    return src


@pytest.mark.parametrize("arch", ["embedding", "norm", "mlp"])
def test_copy_init_is_exact_deep_copy(gpu_lib, arch):
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch=arch, tokens=64, layers=4,
                after=[2, 4], init="copy", seed=3)
    bb = S.backbone(cfg)
    heads = _store(gpu_lib, cfg)
    src = _copy_src(cfg, bb)
    heads.init("copy", copy_src=src)
    torch.cuda.synchronize()
    for i, k in enumerate(cfg.after):
        for name, t in src[i].items():
            assert torch.equal(heads.master[i][name], t.float()), name      # exact widening
            if not name.startswith("g_"):
                assert torch.equal(heads.operand[i][name], t), name         # bitwise operand
            assert heads.master[i][name].data_ptr() != t.data_ptr()         # deep copy
    # oracle's init_copy selects the same modules (structure)
    bb64 = {"final_norm": to_f64(bb["final_norm"]), "w_out": to_f64(bb["w_out"]),
            "layers": [None] * cfg.layers}
    for k, L in bb["layers"].items():
        bb64["layers"][k - 1] = {n: to_f64(v) for n, v in L.items()}
    for i, k in enumerate(cfg.after):
        po = O.init_copy(arch, bb64, k)
        for name, v in po.items():
            np.testing.assert_array_equal(to_f64(heads.master[i][name]), v)


def test_copy_init_missing_source_is_structure_error(gpu_lib):
    cfg = S.Cfg(name="small", hidden=128, vocab=512, ffn=256, arch="mlp", tokens=64, layers=4,
                after=[2], init="copy", seed=3)
    heads = _store(gpu_lib, cfg)
    src = _copy_src(cfg, S.backbone(cfg))
    del src[0]["w_down"]
    with pytest.raises(gpu_lib.EEError) as e:
        heads.init("copy", copy_src=src)
    assert e.value.code == 6


def test_P7_copy_init_reproduces_original_head(gpu_lib):
    """Tiny config: the Norm exit at the last layer, Copy-initialised, gives the
    original model's loss (oracle's original_final_logits), and the same GPU
    result as feeding the backbone's own head tensors (bitwise)."""
    cfg = S.get_cfg("tiny")
    bb = S.backbone(cfg)
    heads = _store(gpu_lib, cfg, cfg.tokens)
    heads.init("copy", copy_src=_copy_src(cfg, bb))
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg, ignore_frac=0.0)
    loss = heads.step([h.cuda() for h in hidden], targets.cuda()).clone()
    torch.cuda.synchronize()
    # original head on the last hidden state (exit 2 sits after the last layer L=2)
    bb64 = {"final_norm": to_f64(bb["final_norm"]), "w_out": to_f64(bb["w_out"])}
    Sorig = O.original_final_logits(bb64, to_f64(hidden[1]), 1e-5)
    st = O.lm_loss_stats(Sorig, targets.numpy())
    L_orig = float(st["loss"].mean())
    assert abs(loss[1].item() - L_orig) / L_orig <= 1e-3
    # feeding the backbone tensors directly as params gives a bitwise-equal loss
    p = [{"w_out": bb["w_out"].float(), "g_f": bb["final_norm"].float()}] * 2
    l2, _, _, _ = gpu_step(gpu_lib, cfg, hidden, targets, p, [1.0, 1.0])
    assert torch.equal(l2[1], loss[1])


def test_P15_random_init_statistics_and_determinism(gpu_lib):
    cfg = S.Cfg(name="small", hidden=256, vocab=4096, ffn=512, arch="mlp", tokens=64, layers=2,
                after=[1, 2], init="random", seed=0)
    a, b, c = _store(gpu_lib, cfg), _store(gpu_lib, cfg), _store(gpu_lib, cfg)
    a.init("random", seed=1234, std=0.02)
    b.init("random", seed=1234, std=0.02)
    c.init("random", seed=1235, std=0.02)
    torch.cuda.synchronize()
    for i in range(2):
        for k in ("w_gate", "w_up", "w_down", "w_out"):
            t = a.master[i][k]
            assert t.numel() >= 10_000
            assert 0.018 <= t.std().item() <= 0.022, (k, t.std().item())
            assert abs(t.mean().item()) < 1e-3
            assert torch.equal(t, b.master[i][k])                       # same seed: bitwise
            assert not torch.equal(t, c.master[i][k])                   # different seed
            assert torch.equal(a.operand[i][k], t.to(torch.bfloat16))
        assert torch.all(a.master[i]["g_a"] == 1) and torch.all(a.master[i]["g_f"] == 1)
    # different exits / tensors draw different streams
    assert not torch.equal(a.master[0]["w_gate"], a.master[1]["w_gate"])
    assert not torch.equal(a.master[0]["w_gate"], a.master[0]["w_up"])
    # normality: fraction within 1 sigma ~ 0.6827
    t = a.master[0]["w_out"].flatten()
    frac = ((t.abs() <= 0.02).float().mean()).item()
    assert abs(frac - 0.6827) < 0.01


def test_adam_matches_oracle_and_zero_grad(gpu_lib):
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300, layers=2,
                after=[1, 2], init="random", seed=4)
    heads = _store(gpu_lib, cfg, 300)
    heads.init("random", seed=7)
    hidden = [h.cuda() for h in S.hidden_states(cfg, 300)]
    targets = S.targets(cfg, 300).cuda()
    theta0 = [{k: v.clone() for k, v in m.items()} for m in heads.master]
    ms = [{k: torch.zeros_like(v) for k, v in m.items()} for m in heads.master]
    vs = [{k: torch.zeros_like(v) for k, v in m.items()} for m in heads.master]
    for it in range(1, 4):
        heads.step(hidden, targets, exit_weights=[1.0, 0.0])       # exit 2: alpha = 0
        g = [{k: v.clone() for k, v in gd.items()} for gd in heads.grads]
        lr = gpu_lib.ee_lr_at(it, 100)
        heads.adam(lr)
        torch.cuda.synchronize()
        for i in range(2):
            for k in g[i]:
                th, m, v = O.adam_update(to_f64(theta0[i][k]), to_f64(g[i][k]), to_f64(ms[i][k]),
                                         to_f64(vs[i][k]), lr, 0.9, 0.95, 1e-5, 0.0, it)
                np.testing.assert_allclose(to_f64(heads.master[i][k]), th, rtol=1e-6, atol=1e-9)
                theta0[i][k] = heads.master[i][k].clone()
                ms[i][k] = torch.from_numpy(m).float().cuda()
                vs[i][k] = torch.from_numpy(v).float().cuda()
                if not k.startswith("g_"):
                    assert torch.equal(heads.operand[i][k], heads.master[i][k].to(torch.bfloat16))
    # exit 2 had alpha = 0 throughout: bitwise unchanged
    fresh = _store(gpu_lib, cfg, 1)
    fresh.init("random", seed=7)
    for k in heads.master[1]:
        assert torch.equal(heads.master[1][k], fresh.master[1][k]), k


def test_sgd_step_decreases_loss(gpu_lib):
    """A few SGD steps on the same batch reduce every exit's loss."""
    cfg = S.get_cfg("tiny")
    heads = _store(gpu_lib, cfg, cfg.tokens)
    heads.init("copy", copy_src=_copy_src(cfg, S.backbone(cfg)))
    hidden = [h.cuda() for h in S.hidden_states(cfg)]
    targets = S.targets(cfg).cuda()
    l0 = heads.step(hidden, targets).clone()
    for _ in range(5):
        heads.step(hidden, targets)
        gpu_lib.ee_sgd_update(heads.cfg, heads.master, heads.operand, heads.grads, lr=0.5)
    l1 = heads.step(hidden, targets).clone()
    torch.cuda.synchronize()
    assert torch.all(l1 < l0), (l0, l1)


def test_per_exit_update_with_shared_grad_buffer_equals_full_step(gpu_lib):
    """Exit-by-exit tune + Adam with one shared gradient buffer ("forward,
    backward, and parameter update for each early-exit layer, without any
    dependency between early exits") gives bitwise the same parameters as
    tuning all exits and then updating them all."""
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300, layers=3,
                after=[1, 2, 3], init="random", seed=41)
    spec = gpu_lib.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, 3, cfg.arch)
    a = gpu_lib.ExitHeads(spec, 300)
    b = gpu_lib.ExitHeads(spec, 300, grad_buffers=1)
    a.init("random", seed=5)
    b.init("random", seed=5)
    hidden = [h.cuda() for h in S.hidden_states(cfg, 300)]
    targets = S.targets(cfg, 300).cuda()
    for it in range(2):
        la = a.step(hidden, targets).clone()
        a.adam(1e-3)
        lb = b.step_per_exit(hidden, targets, 1e-3).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, lb)
    for i in range(3):
        for k in a.master[i]:
            assert torch.equal(a.master[i][k], b.master[i][k]), (i, k)
            assert torch.equal(a.m[i][k], b.m[i][k]), (i, k)


def test_step_host_streaming_equals_device_step(gpu_lib):
    """Host-resident hidden states streamed per exit (H2D overlapped with the
    previous exit's compute) give bitwise the same losses and gradients."""
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300, layers=3,
                after=[1, 2, 3], init="random", seed=42)
    spec = gpu_lib.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, 3, cfg.arch)
    a = gpu_lib.ExitHeads(spec, 300)
    a.init("random", seed=9)
    hidden = S.hidden_states(cfg, 300)
    targets = S.targets(cfg, 300)
    la = a.step([h.cuda() for h in hidden], targets.cuda()).clone()
    ga = [{k: v.clone() for k, v in g.items()} for g in a.grads]
    lb = a.step_host([h.pin_memory() for h in hidden], targets.pin_memory()).clone()
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    for i in range(3):
        for k in ga[i]:
            assert torch.equal(ga[i][k], a.grads[i][k]), (i, k)


@pytest.mark.parametrize("exits", [2, 3])
def test_step_host_back_to_back_calls(gpu_lib, exits):
    """Calls issued back to back without host synchronisation (the next call's
    first exit is staged while the previous call's last exit computes): each
    call's losses equal the device step on the same inputs, bitwise, for
    alternating input sets (a staging-buffer race would mix them)."""
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300,
                layers=exits, after=list(range(1, exits + 1)), init="random", seed=43)
    spec = gpu_lib.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, exits, cfg.arch)
    a = gpu_lib.ExitHeads(spec, 300)
    a.init("random", seed=10)
    sets = [(S.hidden_states(cfg, 300, seed=s), S.targets(cfg, 300, seed=s)) for s in (1, 2)]
    want = [a.step([h.cuda() for h in hs], t.cuda()).clone() for hs, t in sets]
    host = [([h.pin_memory() for h in hs], t.pin_memory()) for hs, t in sets]
    got = []
    for r in range(24):
        hs, t = host[r % 2]
        got.append(a.step_host(hs, t).clone())
    torch.cuda.synchronize()
    for r in range(24):
        assert torch.equal(got[r], want[r % 2]), r


def test_step_host_after_async_device_step(gpu_lib):
    """The first step_host call allocates its staging buffers while a device
    step() whose input tensors were already freed is still queued: the caching
    allocator may hand those blocks to the staging buffers, so the copy stream
    must not write them before the queued step has read them (the round-1
    driver failure).  Fresh objects each round so the first-call path repeats."""
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=300,
                layers=2, after=[1, 2], init="random", seed=44)
    spec = gpu_lib.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, 2, cfg.arch)
    sets = [(S.hidden_states(cfg, 300, seed=s), S.targets(cfg, 300, seed=s)) for s in (1, 2)]
    host = [([h.pin_memory() for h in hs], t.pin_memory()) for hs, t in sets]
    ref = None
    for r in range(6):
        a = gpu_lib.ExitHeads(spec, 300)
        a.init("random", seed=10)
        if ref is None:
            ref = [a.step([h.cuda() for h in hs], t.cuda()).clone() for hs, t in sets]
            torch.cuda.synchronize()
        la = a.step([h.cuda() for h in sets[0][0]], sets[0][1].cuda()).clone()  # inputs freed
        lb = a.step_host(*host[1]).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, ref[0]), r
        assert torch.equal(lb, ref[1]), r
