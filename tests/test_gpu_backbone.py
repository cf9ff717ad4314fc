"""Frozen backbone partial forward (NEXT #3) on the GPU vs the fp64
oracle (Llama-2 pre-norm layers: RoPE, causal GQA attention, SwiGLU MLP)."""

import numpy as np
import pytest
import torch

from eesynth import to_f64
from harness import rel_fro
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


def _layers(L, h, nh, nkv, F, std, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    d = 128

    def r(*shape, s=std):
        return (torch.randn(*shape, generator=g, device="cuda") * s).to(torch.bfloat16)

    out = []
    for _ in range(L):
        out.append({"g_att": (1 + 0.1 * torch.randn(h, generator=g, device="cuda")).float(),
                    "w_q": r(nh * d, h), "w_k": r(nkv * d, h), "w_v": r(nkv * d, h),
                    "w_o": r(h, nh * d), "g_mlp": (1 + 0.1 * torch.randn(h, generator=g, device="cuda")).float(),
                    "w_gate": r(F, h), "w_up": r(F, h), "w_down": r(h, F)})
    return out


@pytest.mark.parametrize("h,nh,nkv,F,T,B,L,exits,std", [
    (256, 2, 1, 512, 128, 2, 3, [1, 3], 0.06),       # GQA, several tiles and sequences
    (256, 2, 2, 384, 192, 1, 2, [2], 0.06),          # MHA, ragged 64-tiles of the causal loop
    (5120, 40, 40, 13824, 128, 1, 1, [1], 0.02),     # Llama-2-13B layer shape
    (8192, 64, 8, 28672, 64, 1, 1, [1], 0.02),       # Llama-2-70B layer shape (GQA 8)
])
def test_backbone_forward_matches_oracle(gpu_lib, h, nh, nkv, F, T, B, L, exits, std):
    ee = gpu_lib
    n = T * B
    layers = _layers(L, h, nh, nkv, F, std, seed=h + L)
    g = torch.Generator(device="cuda").manual_seed(7)
    x0 = torch.randn(n, h, generator=g, device="cuda").to(torch.bfloat16)
    cfg = ee.make_backbone_config(h, nh, nkv, F, T)
    ws = torch.zeros(ee.ee_backbone_workspace_size(cfg, n), dtype=torch.uint8, device="cuda")
    outs = [torch.zeros(n, h, dtype=torch.bfloat16, device="cuda") for _ in exits]
    ee.ee_backbone_forward(cfg, layers, x0, exits, outs, ws)
    torch.cuda.synchronize()
    l64 = [{k: to_f64(v) for k, v in lay.items()} for lay in layers]
    ref = O.backbone_forward(l64, to_f64(x0), T, nh, nkv, exits, 1e-5)
    x0_64 = to_f64(x0)
    for got, want in zip(outs, ref):
        g64 = to_f64(got)
        upd = rel_fro(g64 - x0_64, want - x0_64)        # the layers' contribution
        full = rel_fro(g64, want)
        print("backbone rel err: update", upd, "full", full)
        assert upd <= 3e-2, (upd, full)
        assert full <= 2e-2, (upd, full)
