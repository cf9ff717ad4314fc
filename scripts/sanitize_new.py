"""Small launches of the r01e kernels for compute-sanitizer (attention tc fwd/bwd,
Layer exit step, skinny decode inference)."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import eesynth as S
import paper_2402_00518_b200 as ee
from harness import gpu_step

ee.load()
# attention, T = 192 (partial tiles), GQA 2:1
T, Hq, Hkv, B = 192, 2, 1, 2
n = B * T
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
k = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
v = torch.randn(n, Hkv * 128, device="cuda", generator=g).bfloat16()
do = torch.randn(n, Hq * 128, device="cuda", generator=g).bfloat16()
o = torch.empty_like(q); lse2 = torch.empty(n, Hq, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
scr = torch.empty(n, Hq, device="cuda")
ee.ee_test_attention(q, k, v, o, lse2, T, Hq, Hkv, dout=do, dq=dq, dk=dk, dv=dv, scratch=scr, impl=1)
torch.cuda.synchronize()
# Layer exit step (tiny_layer)
cfg = S.get_cfg("tiny_layer")
loss, grads, aux, st = gpu_step(ee, cfg, S.hidden_states(cfg), S.targets(cfg), S.head_params(cfg), [1.0, 0.5])
assert st == (0, -1), st
# skinny inference, n = 5 and 13
for nt in (5, 13):
    c = S.Cfg(name="small", hidden=256, vocab=2056, ffn=384, arch="mlp", tokens=nt, layers=2,
              after=[1, 2], init="random", seed=3)
    heads = ee.ExitHeads(ee.HeadSpec(256, 2056, 384, 2, "mlp"), max_tokens=nt, adam=False)
    heads.init("random", seed=2)
    heads.infer([x.cuda() for x in S.hidden_states(c, nt)], 0.5)
torch.cuda.synchronize()
print("sanitize run ok")
