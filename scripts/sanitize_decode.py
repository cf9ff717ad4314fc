"""Decode-shape exit heads (skinny.cu: TMA ring, stream-K fix-up, PDL chain) at
sizes whose (row block, k chunk) units outnumber the CTAs, for compute-sanitizer
(memcheck / racecheck / synccheck)."""
import os
import sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import eesynth as S
import paper_2402_00518_b200 as ee

ee.load()
for arch, h, V, F, nt in (("mlp", 1088, 4104, 2944, 1), ("mlp", 1088, 4104, 2944, 13),
                          ("norm", 2048, 8008, 0, 16), ("embedding", 1024, 4104, 0, 3)):
    c = S.Cfg(name="small", hidden=h, vocab=V, ffn=F, arch=arch, tokens=nt, layers=2,
              after=[1, 2], init="random", seed=3)
    heads = ee.ExitHeads(ee.HeadSpec(h, V, F, 2, arch), max_tokens=nt, adam=False)
    heads.init("random", seed=2)
    heads.infer([x.cuda() for x in S.hidden_states(c, nt)], 0.5)
torch.cuda.synchronize()
print("sanitize decode ok")
