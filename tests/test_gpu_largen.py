"""Gradient parity at token counts that take the bench's GEMM code paths.

The weight-gradient GEMMs contract over the token axis, so with N >= 16384
they take the long-K static schedule with the per-wave barrier
(csrc/gemm.cu launch2), and the activation GEMMs (a2, a8, a12 du) see
hundreds of CTA-pair tiles under the dynamic tile scheduler; the EPI_F32T
transposed stores run over several waves.  h, V and F are kept small enough
for the fp64 oracle to finish in seconds but large enough that the long-K
weight-gradient GEMMs span more than one wave of 74 CTA pairs (dW_gate|up at
h 1024, F 4096: 4 x 32 = 128 pair tiles), with ragged token and vocab tails.
Every gradient tensor is compared with the oracle at the north_star bound
(relative Frobenius <= 2e-2) and the loss at 1e-3, for both ds_modes
(§2.2: backprop into the exit parameters only).
"""

import numpy as np
import pytest

import eesynth as S
from harness import GRAD_RTOL, grad_rtol, LOSS_RTOL, gpu_step, oracle_exit, rel_fro

pytestmark = pytest.mark.gpu


def _check(ee, cfg, n, ds_mode, attn=None):
    hidden = S.hidden_states(cfg, n, seed=5)
    targets = S.targets(cfg, n, seed=5)
    params = S.head_params(cfg, seed=5)
    loss, grads, aux, status = gpu_step(ee, cfg, hidden, targets, params, [0.75],
                                        ds_mode=ds_mode)
    assert status == (0, -1), status
    res = oracle_exit(cfg.arch, params[0], hidden[0], targets, 0.75, attn=attn)
    lrel = abs(loss[0].item() - res.loss) / res.loss
    errs = {k: rel_fro(grads[0][k].double().cpu().numpy(), g) for k, g in res.grads.items()}
    print(f"{cfg.arch} n={n} {ds_mode}: loss_rel {lrel:.2e}",
          {k: f"{e:.2e}" for k, e in errs.items()})
    assert lrel <= LOSS_RTOL, (loss[0].item(), res.loss)
    for k, e in errs.items():
        assert e <= grad_rtol(cfg.arch, k), (k, e)
    # per-token loss on every row (not a sample): a tile lost by the scheduler
    # would leave NaN / garbage rows here
    lt = aux[0]["loss_tok"].double().cpu().numpy()
    ref = res.stats["loss"]
    assert np.max(np.abs(lt - ref)) <= 2e-2 * max(1.0, float(np.max(np.abs(ref))))


@pytest.mark.parametrize("ds_mode", ["recompute", "stored_p"])
def test_mlp_exit_long_k_multiwave(gpu_lib, ds_mode):
    cfg = S.Cfg(name="largen", hidden=1024, vocab=4104, ffn=4096, arch="mlp", tokens=16461,
                layers=1, after=[1], init="random", seed=21)
    _check(gpu_lib, cfg, 16461, ds_mode)


@pytest.mark.parametrize("ds_mode", ["recompute", "stored_p"])
def test_norm_exit_long_k(gpu_lib, ds_mode):
    cfg = S.Cfg(name="largen", hidden=2048, vocab=8200, ffn=0, arch="norm", tokens=16411,
                layers=1, after=[1], init="random", seed=22)
    _check(gpu_lib, cfg, 16411, ds_mode)


def test_layer_exit_t2048(gpu_lib):
    """Layer exit on 8 sequences of T = 2048 (GQA 4:2): the attention
    kernels at the paper's sequence length and the long-K weight gradients."""
    cfg = S.Cfg(name="largen", hidden=512, vocab=4104, ffn=1024, arch="layer", tokens=8 * 2048,
                layers=1, after=[1], init="random", seed=23, n_heads=4, n_kv_heads=2,
                seq_len=2048)
    _check(gpu_lib, cfg, cfg.tokens, "recompute", attn=S.attn_geometry(cfg))
