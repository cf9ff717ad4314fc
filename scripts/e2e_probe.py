"""Where does the 7B end-to-end step lose time?  device step vs step_host vs H2D alone."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eesynth as S
import paper_2402_00518_b200 as ee

cfg = S.get_cfg(sys.argv[1] if len(sys.argv) > 1 else "7b")
ee.load()
dev = torch.device("cuda")
heads = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch), cfg.tokens)
heads.init("random")
hidden = S.hidden_states(cfg, cfg.tokens, device=dev)
targets = S.targets(cfg, cfg.tokens, device=dev)
h_host = [h.cpu().pin_memory() for h in hidden]
t_host = targets.cpu().pin_memory()
print("pinned:", [h.is_pinned() for h in h_host], t_host.is_pinned())

def timeit(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n, (time.perf_counter() - t0) * 1e3 / n

print("device step+adam", timeit(lambda: (heads.step(hidden, targets), heads.adam(1e-4))))
print("step_host+adam", timeit(lambda: (heads.step_host(h_host, t_host), heads.adam(1e-4))))
print("step_host only", timeit(lambda: heads.step_host(h_host, t_host)))
print("H2D only", timeit(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(hidden, h_host)]))
loss_host = torch.empty(cfg.exits).pin_memory()
print("step_host+adam+loss D2H", timeit(lambda: (heads.step_host(h_host, t_host), heads.adam(1e-4), loss_host.copy_(heads.loss, non_blocking=True))))
