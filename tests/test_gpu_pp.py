"""Forward-communication-only pipeline schedule (NEXT #3) through
the CUDA kernels on one GPU: 2 backbone stages x 2 microbatches, each stage
running ee_backbone_forward on its layers and ee_tune_step on its own exits
right after (gradients accumulated over microbatches, global valid count);
the activation crosses the stage boundary in bf16 through a channel (the
NCCL/gloo transport itself is tests/test_pp_gloo.py).  Equals the
single-process run (full backbone, all exits, full batch) within the
north_star tolerances, and is anchored to the fp64 oracle: the hidden states
each stage hands its exit match oracle.backbone_forward (the partial forward of
P:260; test_gpu_backbone's bound), and each stage's accumulated loss and
gradients match oracle.exit_loss_and_grads on exactly those hidden states over
the full batch with the global valid count (north_star bounds)."""

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from harness import GRAD_RTOL, LOSS_RTOL, oracle_exit, rel_fro
from oracle import ee_oracle as O
from test_gpu_backbone import _layers

pytestmark = pytest.mark.gpu


def test_pipeline_forward_only_two_stages(gpu_lib):
    from paper_2402_00518_b200.parallel import pipeline_forward_only_step
    ee = gpu_lib
    h, nh, nkv, F, T, V = 256, 2, 1, 384, 128, 1000
    n_layers, micro, mb = 4, 2, 2 * T                  # 2 microbatches of 2 sequences
    N = micro * mb
    layers = _layers(n_layers, h, nh, nkv, F, 0.06, seed=5)
    bcfg = ee.make_backbone_config(h, nh, nkv, F, T)
    cfg = S.Cfg(name="small", hidden=h, vocab=V, ffn=F, arch="mlp", tokens=N, layers=n_layers,
                after=[2, 4], init="random", seed=9)
    params = S.head_params(cfg)
    x0 = S.hidden_states(cfg, N)[0].cuda()
    targets = S.targets(cfg, N).cuda()
    W = torch.tensor([int((targets != -1).sum())], dtype=torch.int64, device="cuda")

    # ---- reference: one process, full backbone, both exits, full batch
    hid = [torch.empty(N, h, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    ws = torch.zeros(ee.ee_backbone_workspace_size(bcfg, N), dtype=torch.uint8, device="cuda")
    ee.ee_backbone_forward(bcfg, layers, x0, [2, 4], hid, ws)
    spec = ee.HeadSpec(h, V, F, 2, "mlp")
    ref = ee.ExitHeads(spec, N, adam=False)
    for i in range(2):
        for k, v in params[i].items():
            ref.master[i][k].copy_(v)
            if not k.startswith("g_"):
                ref.operand[i][k].copy_(v.to(torch.bfloat16))
    ref_loss = ref.step(hid, targets).clone()

    # ---- pipeline: stage s owns layers [2s+1, 2s+2] and the exit after layer 2s+2
    channel = []
    stage_loss, stage_grads = [], []
    captured = [[], []]
    for stage in range(2):
        heads = ee.ExitHeads(ee.HeadSpec(h, V, F, 1, "mlp"), mb, adam=False)
        for k, v in params[stage].items():
            heads.master[0][k].copy_(v)
            if not k.startswith("g_"):
                heads.operand[0][k].copy_(v.to(torch.bfloat16))
        wsb = torch.zeros(ee.ee_backbone_workspace_size(bcfg, mb), dtype=torch.uint8, device="cuda")
        my_layers = layers[2 * stage:2 * stage + 2]
        out = {}
        total = torch.zeros(1, device="cuda")

        def fwd(m, x_in):
            x = x0[m * mb:(m + 1) * mb].contiguous() if x_in is None else x_in
            y = torch.empty(mb, h, dtype=torch.bfloat16, device="cuda")
            ee.ee_backbone_forward(bcfg, my_layers, x, [2], [y], wsb)
            out[m] = y                                  # this stage's exit sits after its last layer
            captured[stage].append(y.clone())
            return y

        def exits(m):
            heads.step([out.pop(m)], targets[m * mb:(m + 1) * mb].contiguous(), accumulate=m > 0,
                       valid_count=W)
            total.add_(heads.loss)

        pipeline_forward_only_step(stage, 2, micro, fwd, exits,
                                   send=lambda m, t: channel.append(t),
                                   recv=lambda m: channel.pop(0))
        torch.cuda.synchronize()
        assert not out
        stage_loss.append(total.item())
        stage_grads.append({k: v.clone() for k, v in heads.grads[0].items()})
    assert not channel
    for i in range(2):
        assert abs(stage_loss[i] - ref_loss[i].item()) <= 1e-3 * abs(ref_loss[i].item())
        for k in stage_grads[i]:
            assert rel_fro(stage_grads[i][k].double().cpu().numpy(),
                           ref.grads[i][k].double().cpu().numpy()) <= 2e-2, (i, k)

    # ---- oracle anchor: the partial forward and each stage's exit
    l64 = [{k: to_f64(v.cpu()) for k, v in L.items()} for L in layers]
    want_h = O.backbone_forward(l64, to_f64(x0.cpu()), T, nh, nkv, [2, 4], 1e-5)
    tg = targets.cpu()
    for s_ in range(2):
        got_h = torch.cat(captured[s_]).cpu()
        assert rel_fro(to_f64(got_h), want_h[s_]) <= 2e-2, s_
        res = oracle_exit("mlp", params[s_], got_h, tg, 1.0)
        assert abs(stage_loss[s_] - res.loss) <= LOSS_RTOL * res.loss, (s_, stage_loss[s_], res.loss)
        for k, g in res.grads.items():
            e = rel_fro(stage_grads[s_][k].double().cpu().numpy(), g)
            assert e <= GRAD_RTOL, (s_, k, e)
