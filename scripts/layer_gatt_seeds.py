"""Single-GPU Layer-exit gradient errors vs the oracle over seeds (tiny_layer,
512 tokens): how close the gain gradients sit to the north_star bound."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import eesynth as S
import paper_2402_00518_b200 as ee
from harness import gpu_step, oracle_exit, rel_fro
ee.load()
for seed in range(56, 72):
    cfg = S.get_cfg("tiny_layer", seed=seed)
    cfg.tokens = 512
    hidden = S.hidden_states(cfg); targets = S.targets(cfg); params = S.head_params(cfg)
    loss, grads, aux, st = gpu_step(ee, cfg, hidden, targets, params, [1.0, 0.5])
    for i in range(2):
        res = oracle_exit("layer", params[i], hidden[i], targets, [1.0, 0.5][i], attn=S.attn_geometry(cfg))
        e = {k: rel_fro(grads[i][k].double().cpu().numpy(), g) for k, g in res.grads.items()}
        worst = max(e, key=e.get)
        print(seed, i, worst, f"{e[worst]:.2e}", f"g_att {e['g_att']:.2e} g_a {e['g_a']:.2e} g_f {e['g_f']:.2e}", flush=True)
