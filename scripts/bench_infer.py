"""Confidence-based early-exit decision at decode shapes (NEXT #4):
ee_exit_infer over all exits for M = batch tokens, 70B-shaped MLP heads.
Latency-bound: every exit head's weights are streamed once per call, so the
roofline is HBM bytes / measured copy bandwidth."""
import json
import sys

import torch

sys.path.insert(0, ".")
import eesynth as S
import paper_2402_00518_b200 as ee

peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}
hbm = peaks.get("hbm_gbs")
cfg = S.get_cfg(sys.argv[1] if len(sys.argv) > 1 else "70b")
h, V, F, E = cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits
heads = ee.ExitHeads(ee.HeadSpec(h, V, F, E, cfg.arch), max_tokens=4096, adam=False)
heads.init("random", seed=1)
w_bytes = 2 * (V * h + (3 * F * h if cfg.arch == "mlp" else 0))   # bf16 operands per exit
Ms = [int(v) for v in __import__('os').environ.get('EE_INFER_M', '1,8,16,64,512').split(',')]
reps = int(__import__('os').environ.get('EE_INFER_REPS', '10'))
for M in Ms:
    hidden = [x.cuda() for x in S.hidden_states(cfg, M)]
    for _ in range(3):
        heads.infer(hidden, 0.9)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        heads.infer(hidden, 0.9)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    byt = E * (w_bytes + 2 * M * h)
    print(json.dumps({"config": cfg.name, "exits": E, "batch_tokens": M, "ms": round(ms, 4),
                      "hbm_bytes": byt, "GB_s": round(byt / ms / 1e6, 1),
                      "frac_of_hbm": (round(byt / ms / 1e6 / hbm, 3) if hbm else None)}), flush=True)
