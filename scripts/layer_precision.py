"""Investigation: Layer-exit gradient error vs attention peakedness and
residual outlier channels (which bf16 rounding dominates)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
import eesynth as S
from harness import gpu_step, oracle_exit, rel_fro
import paper_2402_00518_b200 as ee

ee.load()
base = dict(hidden=512, vocab=2056, ffn=640, n_heads=4, n_kv_heads=1, seq_len=192, tokens=384)
orig_attn = S._attn_params
for qk_mult in (2.0, 1.0, 0.5):
    for massive in (50.0, 1.0):
        S.MASSIVE_SCALE = massive
        def ap(cfg, g, device, m=qk_mult):
            p = orig_attn(cfg, g, device)
            p["w_q"] = p["w_q"] * (m / 2.0)
            p["w_k"] = p["w_k"] * (m / 2.0)
            return p
        S._attn_params = ap
        for seed in (8, 9):
            cfg = S.get_cfg("tiny_layer", seed=seed, **base)
            hidden, targets, params = S.hidden_states(cfg), S.targets(cfg), S.head_params(cfg)
            loss, grads, aux, st = gpu_step(ee, cfg, hidden, targets, params, [1.0, 0.5])
            errs = []
            for i in range(2):
                res = oracle_exit("layer", params[i], hidden[i], targets, [1.0, 0.5][i],
                                  attn=S.attn_geometry(cfg))
                errs.append({k: round(rel_fro(grads[i][k].double().cpu().numpy(), g), 4)
                             for k, g in res.grads.items() if k in ("g_att", "w_q", "w_k", "w_v", "w_o", "g_a")})
            print(f"qk={qk_mult} massive={massive} seed={seed}", errs, flush=True)
