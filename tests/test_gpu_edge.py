"""Edge cases on the GPU: empty batches, a single token, the smallest legal
shapes (h = 64, V = 8, F = 128), a single minimal Layer sequence (T = 64),
and empty inference -- against the oracle or the contract in include/ee.h."""

import numpy as np
import pytest
import torch

import eesynth as S
from harness import attn_kwargs, compare_exit, gpu_step, oracle_exit

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch", ["embedding", "norm", "mlp", "layer"])
def test_empty_batch_zeroes_grads_and_loss(gpu_lib, arch):
    ee = gpu_lib
    cfg = S.get_cfg("tiny_layer") if arch == "layer" else S.Cfg(
        name="small", hidden=128, vocab=512, ffn=256, arch=arch, tokens=0, layers=2, after=[1, 2],
        init="random", seed=1)
    params = S.head_params(cfg)
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 2, arch, **attn_kwargs(cfg))
    ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().to(torch.bfloat16))
            for k, v in p.items()} for p in params]
    grads = [{k: torch.full(v.shape, 7.0, device="cuda") for k, v in p.items()} for p in params]
    ws = torch.zeros(max(ee.ee_workspace_size(c, 0), 256), dtype=torch.uint8, device="cuda")
    loss = torch.full((2,), 3.0, device="cuda")
    hid = [torch.zeros(0, cfg.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    ee.ee_tune_step(c, hid, torch.zeros(0, dtype=torch.int32, device="cuda"), [1.0, 1.0], ops,
                    grads, loss, ws)
    torch.cuda.synchronize()
    assert torch.all(loss == 0)
    for g in grads:
        for k, v in g.items():
            assert torch.all(v == 0), k
    # accumulate = 1 leaves the gradients untouched
    g2 = [{k: torch.full(v.shape, 7.0, device="cuda") for k, v in p.items()} for p in params]
    ee.ee_tune_step(c, hid, torch.zeros(0, dtype=torch.int32, device="cuda"), [1.0, 1.0], ops,
                    g2, loss, ws, accumulate=True)
    torch.cuda.synchronize()
    for g in g2:
        for k, v in g.items():
            assert torch.all(v == 7.0), k
    assert ee.ee_get_status(ws) == (0, -1)


@pytest.mark.parametrize("arch,h,V,F,n", [("mlp", 128, 1000, 256, 1), ("norm", 64, 8, 0, 3),
                                          ("mlp", 64, 8, 128, 5), ("embedding", 64, 16, 0, 1)])
def test_single_token_and_minimum_shapes(gpu_lib, arch, h, V, F, n):
    cfg = S.Cfg(name="small", hidden=h, vocab=V, ffn=F, arch=arch, tokens=n, layers=1, after=[1],
                init="random", seed=h + V + n)
    hidden = S.hidden_states(cfg, n)
    targets = S.targets(cfg, n, ignore_frac=0.0)
    params = S.head_params(cfg)
    loss, grads, aux, st = gpu_step(gpu_lib, cfg, hidden, targets, params, [0.7])
    assert st == (0, -1)
    res = oracle_exit(arch, params[0], hidden[0], targets, 0.7)
    compare_exit(arch, res, loss[0].item(), grads[0], aux[0], targets)


def test_layer_exit_single_minimal_sequence(gpu_lib):
    cfg = S.get_cfg("tiny_layer", hidden=128, n_heads=1, n_kv_heads=1, seq_len=64, tokens=64,
                    ffn=128, vocab=64, seed=77)
    cfg.after = cfg.after[:1]
    cfg.exits = 1
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    loss, grads, aux, st = gpu_step(gpu_lib, cfg, hidden, targets, params, [1.0])
    assert st == (0, -1)
    res = oracle_exit("layer", params[0], hidden[0], targets, 1.0, attn=S.attn_geometry(cfg))
    compare_exit("layer", res, loss[0].item(), grads[0], aux[0], targets)


def test_empty_inference(gpu_lib):
    ee = gpu_lib
    c = ee.make_config(128, 512, 256, 2, "mlp")
    cfg = S.Cfg(name="small", hidden=128, vocab=512, ffn=256, arch="mlp", tokens=0, layers=2,
                after=[1, 2], init="random", seed=2)
    ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().to(torch.bfloat16))
            for k, v in p.items()} for p in S.head_params(cfg)]
    ws = torch.zeros(max(ee.ee_workspace_size(c, 0), 256), dtype=torch.uint8, device="cuda")
    e = [torch.zeros(0, dtype=torch.int32, device="cuda")] * 2
    f = [torch.zeros(0, device="cuda")] * 2
    ee.ee_exit_infer(c, [torch.zeros(0, 128, dtype=torch.bfloat16, device="cuda")] * 2, ops, 0.5,
                     e, f, ws, first_exit=torch.zeros(0, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
