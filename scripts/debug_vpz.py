import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2402_00518_b200 as ee
import eesynth as S
import test_gpu_vp_fused as T
ee.load()
cfg = T._cfg("layer", 37)
hidden = S.hidden_states(cfg, 256); targets = S.targets(cfg, 256); params = S.head_params(cfg)
T._run_vp_adam(ee, cfg, 1, hidden, targets, params, sharded=True, steps=1)
for steps in (1,):
    ref = T._run_vp_adam(ee, cfg, 2, hidden, targets, params, sharded=False, steps=steps)
    got = T._run_vp_adam(ee, cfg, 2, hidden, targets, params, sharded=True, steps=steps)
    for r in range(2):
        print("rank", r, "loss", got[r][3].tolist(), ref[r][3].tolist(), got[r][4])
        for i in range(cfg.exits):
            for k, t in ref[r][0][i].items():
                g = got[r][0][i][k]
                if not torch.equal(g, t):
                    d = (g.float() - t.float()).abs()
                    print("  operand differs", i, k, float(d.max()), int((d > 0).sum()), t.numel())
            for k, full in ref[r][1][i].items():
                if k == "w_out":
                    if not torch.equal(got[r][1][i][k], full): print("  w_out master differs", i)
                    continue
                b, rows = got[r][2][k][0], got[r][2][k][1]
                want = full.reshape(-1, full.shape[-1])[b:b + rows]
                if not torch.equal(got[r][1][i][k], want):
                    print("  master differs", i, k, float((got[r][1][i][k]-want).abs().max()))
