"""Layer exits (NEXT #2; P:210 architecture, P:237 Copy init) on the GPU
against the fp64 oracle: loss, every parameter gradient (attention tensors
included), per-token aux, at sizes spanning several GEMM tiles and attention
tiles, GQA and MHA, a ragged vocabulary, and several sequences."""

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from harness import attn_kwargs, compare_exit, gpu_step, oracle_exit
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(**over):
    return S.get_cfg("tiny_layer", **over)


@pytest.mark.parametrize("over", [
    {},                                                                   # GQA 2:1, 2 seqs of 128
    dict(hidden=384, vocab=520, ffn=256, n_heads=3, n_kv_heads=3, seq_len=64, tokens=192,
         seed=7),                                                         # MHA, 3 seqs, ragged V
    dict(hidden=512, vocab=2056, ffn=640, n_heads=4, n_kv_heads=1, seq_len=192, tokens=384,
         seed=8),                                                         # GQA 4:1, T = 3 tiles
])
def test_layer_exit_parity(gpu_lib, over):
    cfg = _cfg(**over)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    alphas = [1.0, 0.5][:cfg.exits]
    loss, grads, aux, st = gpu_step(gpu_lib, cfg, hidden, targets, params, alphas)
    assert st == (0, -1)
    at = S.attn_geometry(cfg)
    for i in range(cfg.exits):
        res = oracle_exit("layer", params[i], hidden[i], targets, alphas[i], attn=at)
        g = {k: v for k, v in grads[i].items()}
        errs = compare_exit("layer", res, loss[i].item(), g, aux[i], targets, tag=f"exit{i}")
        assert set(res.grads) == set(params[i])
        print(i, {k: round(v, 5) if isinstance(v, float) else v for k, v in errs.items()})


def test_layer_exit_accumulate_and_alpha_zero(gpu_lib):
    cfg = _cfg()
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    _, g1, _, _ = gpu_step(gpu_lib, cfg, hidden, targets, params, [1.0, 0.0])
    for k, v in g1[1].items():
        assert torch.all(v == 0), k                                      # alpha = 0: exact zeros
    g2 = [{k: v.clone() for k, v in d.items()} for d in g1]
    _, g2, _, _ = gpu_step(gpu_lib, cfg, hidden, targets, params, [1.0, 0.0], accumulate=True,
                           grads=g2)
    for k in g1[0]:
        torch.testing.assert_close(g2[0][k], 2 * g1[0][k], rtol=1e-6, atol=0)


def test_layer_exit_tokens_must_be_whole_sequences(gpu_lib):
    cfg = _cfg()
    hidden = [h[:200] for h in S.hidden_states(cfg)]
    with pytest.raises(gpu_lib.EEError) as e:
        gpu_step(gpu_lib, cfg, hidden, S.targets(cfg)[:200], S.head_params(cfg), [1.0, 1.0])
    assert e.value.code == 2


def test_layer_copy_init_adam_and_skip_identity(gpu_lib):
    """Copy init copies the LAST backbone layer into every exit; then
     the exit after layer L-1 reproduces the original model on the same
    input: exit loss at h_{L-1} == the original final head's loss at h_L =
    layer_L(h_{L-1}), h_L computed by our own backbone forward."""
    ee = gpu_lib
    cfg = _cfg()
    bb = S.backbone(cfg)
    last = bb["layers"][cfg.layers]
    spec = ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, "layer", n_heads=cfg.n_heads,
                       n_kv_heads=cfg.n_kv_heads, seq_len=cfg.seq_len)
    heads = ee.ExitHeads(spec, cfg.tokens)
    src = [dict(w_out=bb["w_out"].cuda(), g_f=bb["final_norm"].cuda(), g_a=last["mlp_norm"].cuda(),
                **{k: last[k].cuda() for k in ("w_gate", "w_up", "w_down", "g_att", "w_q", "w_k",
                                               "w_v", "w_o")})
           for _ in range(cfg.exits)]
    heads.init("copy", copy_src=src)
    torch.cuda.synchronize()
    for i in range(cfg.exits):
        for k, t in src[i].items():
            assert torch.equal(heads.master[i][k], t.float()), k
    # backbone: one layer = the copied last layer; h_{L-1} = x0 (synthetic)
    x0 = S.hidden_states(cfg)[0].cuda()
    bcfg = ee.make_backbone_config(cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.seq_len)
    lay = {"g_att": last["g_att"].float().cuda(), "g_mlp": last["mlp_norm"].float().cuda(),
           **{k: last[k].cuda() for k in ("w_q", "w_k", "w_v", "w_o", "w_gate", "w_up", "w_down")}}
    hL = torch.empty_like(x0)
    ws = torch.zeros(ee.ee_backbone_workspace_size(bcfg, cfg.tokens), dtype=torch.uint8,
                     device="cuda")
    ee.ee_backbone_forward(bcfg, [lay], x0, [1], [hL], ws)
    targets = S.targets(cfg).cuda()
    loss = heads.step([x0, x0], targets).clone()
    # original final head on h_L = a Norm exit with the final norm and W_out
    ncfg = S.Cfg(name="n", hidden=cfg.hidden, vocab=cfg.vocab, ffn=0, arch="norm",
                 tokens=cfg.tokens, layers=1, after=[1], init="copy", seed=0)
    l_orig, _, _, _ = gpu_step(ee, ncfg, [hL], targets,
                               [{"w_out": bb["w_out"].float(), "g_f": bb["final_norm"].float()}],
                               [1.0])
    torch.cuda.synchronize()
    assert abs(loss[0].item() - l_orig[0].item()) <= 2e-3 * abs(l_orig[0].item())
    assert torch.equal(loss[0], loss[1])                                 # identical exits
    # one Adam step on the GPU == the oracle's update (per tensor)
    g = [{k: v.clone() for k, v in d.items()} for d in heads.grads]
    theta = [{k: v.clone() for k, v in d.items()} for d in heads.master]
    heads.adam(1e-4)
    torch.cuda.synchronize()
    for k in theta[0]:
        th, _, _ = O.adam_update(to_f64(theta[0][k]), to_f64(g[0][k]), 0.0, 0.0, 1e-4, 0.9, 0.95,
                                 1e-5, 0.0, 1)
        np.testing.assert_allclose(to_f64(heads.master[0][k]), th, rtol=1e-6, atol=1e-9,
                                   err_msg=k)
