"""Seeded sweep over exit shapes (ragged token counts, vocab widths that are
multiples of 8 but not of the 256-wide tiles, h from 64 to 512, F from 128 to
640, every arch incl. Layer exits) against the fp64 oracle at the north_star
tolerances: loss, every parameter gradient, argmax (gap rule), per-token
losses of ignored targets exactly 0.  Catches tiling / tail / masking mistakes
that fixed test shapes can miss."""

import numpy as np
import pytest

import eesynth as S
from harness import compare_exit, gpu_step, oracle_exit

pytestmark = pytest.mark.gpu


def _configs(n_cfg=24, seed=2402):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cfg):
        arch = ["embedding", "norm", "mlp", "layer"][i % 4]
        if arch == "layer":
            heads = int(rng.integers(1, 4))
            divs = [d for d in range(1, heads + 1) if heads % d == 0]
            kv = divs[int(rng.integers(0, len(divs)))]
            h = 128 * heads
            T = int(rng.choice([64, 128, 192]))
            n = T * int(rng.integers(1, 3))
        else:
            h = int(rng.integers(1, 9)) * 64
            n = int(rng.integers(1, 700))
            heads, kv, T = 0, 0, 0
        V = int(rng.integers(2, 400)) * 8
        F = int(rng.integers(1, 6)) * 128 if arch in ("mlp", "layer") else 0
        out.append(dict(arch=arch, h=h, V=V, F=F, n=n, heads=heads, kv=kv, T=T, seed=1000 + i))
    return out


@pytest.mark.parametrize("c", _configs(), ids=lambda c: f"{c['arch']}-h{c['h']}-V{c['V']}-F{c['F']}-n{c['n']}")
def test_shape_sweep_vs_oracle(gpu_lib, c):
    cfg = S.Cfg(name="sweep", hidden=c["h"], vocab=c["V"], ffn=c["F"], arch=c["arch"],
                tokens=c["n"], layers=2, after=[1, 2], init="random", seed=c["seed"],
                n_heads=c["heads"], n_kv_heads=c["kv"], seq_len=c["T"])
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg, ignore_frac=0.05)
    params = S.head_params(cfg)
    loss, grads, aux, st = gpu_step(gpu_lib, cfg, hidden, targets, params, [1.0, 0.5])
    assert st == (0, -1), st
    at = S.attn_geometry(cfg)
    for i, a in enumerate([1.0, 0.5]):
        res = oracle_exit(cfg.arch, params[i], hidden[i], targets, a, attn=at)
        compare_exit(cfg.arch, res, loss[i].item(), grads[i], aux[i], targets, tag=f"exit{i}")
