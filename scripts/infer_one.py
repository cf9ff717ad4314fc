"""One ee_exit_infer call at batch 1 (70B heads, 4 MLP exits) for ncu."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import eesynth as S
import paper_2402_00518_b200 as ee
cfg = S.get_cfg("70b")
heads = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch), max_tokens=64, adam=False)
heads.init("random", seed=1)
hidden = [x.cuda() for x in S.hidden_states(cfg, 1)]
for _ in range(3):
    heads.infer(hidden, 0.9)
torch.cuda.synchronize()
