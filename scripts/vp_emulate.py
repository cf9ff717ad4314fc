"""One rank of the vocab-parallel step at P ranks, on one GPU (compute only).

BASELINE configs[3] shards W_out over 8 GPUs (strong scaling: 65 536 tokens
in total).  With one GPU available, this runs rank 0's share of that job
through the product orchestration (vocab_parallel_step_fused): the exit body
on N/P tokens, the vocab phases on the [V/P x h] W_out shard for all N tokens
(ragged tail tiles included), the fused all-gather / reduce-scatter stores
(every peer pointer aliases this rank's own buffers, so the stores land
locally instead of over NVLink), the slot sum, and Adam on this rank's
parameters.  The small collectives (CE statistics, body-gradient all-reduce)
are no-ops.  It measures the per-rank kernels at the sharded shapes; it is not
a multi-GPU measurement (no NVLink traffic, no peer skew).

  python scripts/vp_emulate.py [--config 70b] [--ranks 8] [--steps 5] [--warmup 3]
Prints one JSON line.
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
from paper_2402_00518_b200.parallel import (GpuPhases, LocalComm, PeerBuffers,  # noqa: E402
                                            vocab_parallel_step_fused, vocab_shard)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="70b")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sharded-body", action="store_true",
                    help="ShardedVPHeads: body gradients to owners + sharded Adam")
    a = ap.parse_args()
    ee.load()
    cfg = S.get_cfg(a.config)
    P, N, h, E = a.ranks, cfg.tokens, cfg.hidden, cfg.exits
    n = N // P
    vb, ve = vocab_shard(cfg.vocab, P, 0)
    dev = torch.device("cuda")
    if a.sharded_body:
        from paper_2402_00518_b200.parallel import ShardedVPHeads
        heads = ShardedVPHeads(ee.HeadSpec(h, cfg.vocab, cfg.ffn, E, cfg.arch), N, 0, P,
                               device=dev)
        heads.connect_local([heads] * P)
    else:
        heads = ee.ExitHeads(ee.HeadSpec(h, cfg.vocab, cfg.ffn, E, cfg.arch, vocab_begin=vb,
                                         vocab_end=ve), N, device=dev)
    heads.init("random", seed=1)
    hidden = [x[:n].contiguous() for x in S.hidden_states(cfg, N, device=dev)]
    targets = S.targets(cfg, N, device=dev)
    peer = PeerBuffers(0, P, N, h, device=dev)
    peer._tables([peer.z_all] * P, [peer.slots] * P, [peer.sig] * P)
    # the barrier would wait for P - 1 peers that never arrive: every rank is this one
    phases = GpuPhases(ee, heads.exit_cfg if a.sharded_body else heads.cfg, heads.workspace)
    phases.barrier = lambda pb: None
    bufs = {"key": torch.zeros(N, dtype=torch.int64, device=dev),
            "sums": torch.zeros(N, 2, device=dev)}
    W = torch.zeros(1, dtype=torch.int64, device=dev)
    ee.ee_count_valid(targets, cfg.vocab, W, heads.workspace)

    def step(it):
        if a.sharded_body:
            heads.set_lr(1e-4)
            vocab_parallel_step_fused(phases, LocalComm(), peer, cfg.arch, hidden, targets,
                                      heads.operand, heads.grads, heads.loss, [1.0] * E, W, bufs,
                                      body=heads)
            return
        vocab_parallel_step_fused(phases, LocalComm(), peer, cfg.arch, hidden, targets,
                                  heads.operand, heads.grads, heads.loss, [1.0] * E, W, bufs)
        heads.adam(1e-4)

    for it in range(a.warmup):
        step(it)
    torch.cuda.synchronize()
    ee.ee_profile_start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for it in range(a.steps):
        step(it)
    e1.record()
    torch.cuda.synchronize()
    prof = ee.ee_profile_stop()
    ms = e0.elapsed_time(e1) / a.steps
    kern = {}
    for name, kms, fe, fa, by in prof:
        d = kern.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += kms
    code, idx = heads.status()
    print(json.dumps({
        "what": f"rank 0 of {P}: vocab-parallel fused step, compute only (see docstring)"
                + ("; exit body updated ZeRO-1 style (ShardedVPHeads)" if a.sharded_body else ""),
        "config": a.config, "ranks": P, "tokens_total": N, "tokens_local": n,
        "w_out_shard_rows": ve - vb, "ms_per_step_rank0": ms,
        "projected_job_tokens_per_s_if_comm_hidden": N / (ms / 1e3),
        "status": code,
        "kernels_ms_per_step": {k: round(v[1] / a.steps, 3)
                                for k, v in sorted(kern.items(), key=lambda kv: -kv[1][1])}}))


if __name__ == "__main__":
    main()
