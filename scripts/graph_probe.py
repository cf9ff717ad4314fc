"""Is the tune+Adam step capturable in a CUDA graph, and does replay help?"""
import sys, torch
sys.path.insert(0, ".")
import eesynth as S
import paper_2402_00518_b200 as ee

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
cfg = S.get_cfg(name)
n = cfg.tokens
heads = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch), n)
heads.init("random", seed=1)
hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
targets = S.targets(cfg, n, device="cuda")

def step():
    heads.step(hidden, targets)
    heads.adam(1e-5)

s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()

def timeit(fn, k=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k

eager = timeit(step)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
torch.cuda.synchronize()
graphed = timeit(g.replay)
l_eager = heads.loss.clone()
print(f"{name}: eager {eager:.3f} ms/step, graph replay {graphed:.3f} ms/step ({eager / graphed:.3f}x)")
