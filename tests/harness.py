"""Shared helpers of the parity tests: run the CUDA path (through the C-ABI
binding) and the fp64 oracle on the same seeded inputs and compare them with
the north_star tolerances:

  per-exit loss          relative error <= 1e-3
  parameter gradients    relative Frobenius error <= 2e-2, per tensor
  argmax                 exact wherever the oracle's top-2 logit gap exceeds
                         delta = 1e-2 * max(1, |max logit|) (A9); otherwise one
                         of the near-tied candidates
  target bookkeeping     exact (ignored tokens have loss 0, valid-count W exact)
"""

from __future__ import annotations

import numpy as np
import torch

from eesynth import to_f64
from oracle import ee_oracle as O

LOSS_RTOL = 1e-3
GRAD_RTOL = 2e-2
# Layer exits (NEXT #2) only: the pre-attention gain's gradient sits at the
# error floor of bf16 GEMM operands -- the fp64 emulation with nothing but the
# kernel's bf16 roundings reaches 1.5-3.0e-2 on it (A27,
# tests/test_bf16_floor.py) -- so its bound is 5e-2 (every other tensor 2e-2).
LAYER_GAIN_RTOL = 5e-2


def grad_rtol(arch, k):
    return LAYER_GAIN_RTOL if (arch == "layer" and k == "g_att") else GRAD_RTOL
TENSORS = ("g_a", "w_gate", "w_up", "w_down", "g_f", "w_out", "g_att", "w_q", "w_k", "w_v", "w_o")


def attn_kwargs(cfg):
    """make_config keywords for the Layer exit's attention geometry."""
    if cfg.arch != "layer":
        return {}
    return dict(n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads,
                seq_len=cfg.seq_len)


def gpu_step(ee, cfg, hidden, targets, params, exit_weights, accumulate=False, grads=None,
             eps=1e-5, weighting="uniform", ds_mode="recompute"):
    """Run ee_tune_step on the GPU.  hidden: list of bf16 tensors (any device);
    params: list of dicts of fp32 tensors (matrices are cast to bf16 operands).
    Returns (loss[E] tensor, grads list of dicts (device fp32), aux list)."""
    E = len(hidden)
    n = targets.numel()
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch, eps,
                       token_weighting=weighting, ds_mode=ds_mode, **attn_kwargs(cfg))
    hid = [h.cuda().contiguous() for h in hidden]
    tg = targets.cuda().to(torch.int32).contiguous()
    ops = [{k: (v.cuda().float().contiguous() if k.startswith("g_") else
                v.cuda().to(torch.bfloat16).contiguous()) for k, v in p.items()} for p in params]
    if grads is None:
        grads = [{k: torch.full(v.shape, float("nan"), device="cuda") for k, v in p.items()}
                 for p in params]
    aux = [{"lse": torch.zeros(n, device="cuda"), "loss_tok": torch.zeros(n, device="cuda"),
            "argmax": torch.zeros(n, dtype=torch.int32, device="cuda"),
            "conf": torch.zeros(n, device="cuda")} for _ in range(E)]
    ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
    loss = torch.full((E,), float("nan"), device="cuda")
    ee.ee_tune_step(c, hid, tg, exit_weights, ops, grads, loss, ws, accumulate=accumulate, aux=aux)
    torch.cuda.synchronize()
    code, idx = ee.ee_get_status(ws)
    return loss, grads, aux, (code, idx)


def oracle_exit(arch, params, hidden, targets, alpha, eps=1e-5, weighting="uniform", attn=None):
    """fp64 oracle on the same bytes (bf16/fp32 inputs widened exactly)."""
    p64 = {k: to_f64(v) for k, v in params.items()}
    return O.exit_loss_and_grads(arch, p64, to_f64(hidden), targets.cpu().numpy().astype(np.int64),
                                 float(alpha), eps, keep_act=True, weighting=weighting, attn=attn)


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def check_argmax(gpu_argmax, S, valid_rows=None):
    """Exact under the gap rule (A9); near ties must pick a tied candidate."""
    gpu_argmax = np.asarray(gpu_argmax)
    srt = np.sort(S, axis=1)
    m = srt[:, -1]
    gap = m - srt[:, -2]
    delta = 1e-2 * np.maximum(1.0, np.abs(m))
    exact = np.argmax(S, axis=1)
    clear = gap > delta
    assert np.array_equal(gpu_argmax[clear], exact[clear]), \
        f"argmax mismatch on {np.sum(gpu_argmax[clear] != exact[clear])} clear rows"
    for r in np.nonzero(~clear)[0]:
        assert S[r, gpu_argmax[r]] >= m[r] - delta[r], f"row {r}: argmax not a near-tie candidate"
    return int(np.sum(clear)), int(np.sum(~clear))


def compare_exit(arch, res, loss_gpu, grads_gpu, aux_gpu, targets, tag=""):
    """Assert north_star tolerances for one exit; returns a dict of errors."""
    out = {}
    L = float(loss_gpu)
    out["loss_rel"] = abs(L - res.loss) / max(abs(res.loss), 1e-30)
    assert out["loss_rel"] <= LOSS_RTOL, (tag, L, res.loss)
    for k, g in res.grads.items():
        e = rel_fro(grads_gpu[k].double().cpu().numpy(), g)
        out[f"grad_{k}"] = e
        assert e <= grad_rtol(arch, k), (tag, k, e)
    t = targets.cpu().numpy()
    valid = t != -1
    lse = aux_gpu["lse"].double().cpu().numpy()
    assert np.max(np.abs(lse - res.stats["lse"])) <= 5e-2, tag
    lt = aux_gpu["loss_tok"].double().cpu().numpy()
    assert np.all(lt[~valid] == 0.0), tag                       # ignored tokens: exactly 0
    out["lse_max_abs"] = float(np.max(np.abs(lse - res.stats["lse"])))
    conf = aux_gpu["conf"].double().cpu().numpy()
    assert np.max(np.abs(conf - res.stats["conf"])) <= 2e-2, tag
    out["argmax_clear"], out["argmax_near"] = check_argmax(aux_gpu["argmax"].cpu().numpy(),
                                                           res.act["S"])
    return out
