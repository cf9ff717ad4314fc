"""One rank of the fused data-parallel step (ShardedDPHeads, ZeRO-1) at P ranks
on one GPU (compute only): the rank's own tokens (--strong: the config's
global tokens / P, the bench default; else all of them: weak scaling), the
gradient rows scattered by the weight-gradient epilogues (every peer pointer
aliases this rank's own arena, so the stores land locally instead of over
NVLink), the sharded Adam over 1/P of the parameters with its operand stores
(P copies into the same local tensors).  Barriers and the two small
all-reduces are no-ops.  Measures the per-rank kernels, not NVLink.

  python scripts/dp_emulate.py [--config 70b_dp] [--ranks 8] [--strong]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import eesynth as S  # noqa: E402
import paper_2402_00518_b200 as ee  # noqa: E402
from paper_2402_00518_b200.parallel import ShardedDPHeads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="70b")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--strong", action="store_true")
    a = ap.parse_args()
    ee.load()
    cfg = S.get_cfg(a.config)
    P, E = a.ranks, cfg.exits
    N = cfg.tokens // P if a.strong else cfg.tokens
    dev = torch.device("cuda")
    heads = ShardedDPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch), N, 0, P,
                           device=dev)
    heads.connect_local([heads] * P)
    heads.barrier = lambda stream=None: None     # every "peer" is this rank
    heads.init("random", seed=1)
    hidden = S.hidden_states(cfg, N, device=dev)
    targets = S.targets(cfg, N, device=dev)
    for _ in range(a.warmup):
        heads.step(hidden, targets, 1e-4)
    torch.cuda.synchronize()
    ee.ee_profile_start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.steps):
        heads.step(hidden, targets, 1e-4)
    e1.record()
    torch.cuda.synchronize()
    prof = ee.ee_profile_stop()
    ms = e0.elapsed_time(e1) / a.steps
    kern = {}
    for name, kms, fe, fa, by in prof:
        kern[name] = kern.get(name, 0.0) + kms
    print(json.dumps({
        "what": f"rank 0 of {P}: fused DP (ZeRO-1) step, compute only (see docstring)",
        "config": a.config, "ranks": P, "tokens_per_rank": N, "ms_per_step_rank0": ms,
        "scaling": "strong" if a.strong else "weak",
        "projected_job_tokens_per_s_if_comm_hidden": P * N / (ms / 1e3),
        "status": heads.status(),
        "kernels_ms_per_step": {k: round(v / a.steps, 3)
                                for k, v in sorted(kern.items(), key=lambda kv: -kv[1])[:12]}}))


if __name__ == "__main__":
    main()
