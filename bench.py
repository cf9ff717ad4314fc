#!/usr/bin/env python
"""bench.py -- EE-Tuning exit-head tuning step on B200 (BASELINE.json metric).

One "step" = one pass of the whole hot path: for every
exit, the exit-head forward, softmax cross-entropy, backward into the exit
parameters, plus the Adam update of all exit parameters.

Default workload at EVERY N (strong scaling, so the driver's per-N values
compare): BASELINE.json configs[4] / SURVEY C4, `70b_dp` -- 70B-shaped heads
(h 8192, V 32000, F 28672), 8 MLP exits at layers 10..80, 65 536 global tokens
(32 x 2048) split over the N ranks, unsharded W_out; synthetic seeded inputs
(eesynth), Copy init from a synthetic backbone.  The step is the fused
data-parallel path (parallel.ShardedDPHeads: gradient reduce-scatter fused into
the weight-gradient GEMM epilogues over CUDA-IPC peer memory, sharded Adam
whose operand stores are the all-gather, ZeRO-1) at every N, N = 1 included.
dS is recomputed (ds_mode "recompute": no [tokens x vocab] matrix in HBM);
the stored-P~ ablation (A24) is timed beside it at N = 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 70b_dp|70b|13b|7b|13b_layer] [--parallel dp|vp]
                  [--scaling strong|weak] [--ds-mode recompute|stored_p]

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script
under torch.distributed.run with N ranks (127.0.0.1); under torchrun --gpus
must equal WORLD_SIZE.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "exit-head tuning tokens/s and % bf16 tensor-core peak at 1/2/4/8 B200"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return dict(PEAKS_FALLBACK, source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms in a thread."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(rows[0][1]), "samples": len(rows),
                "power_w_max": max((num(r[2]) or 0) for r in rows), "reasons": reasons}


def step_flops(cfg, n):
    """Algorithmic FLOPs of one step: 6hV per token per exit
    (Embedding exits have no dz GEMM: 4hV), +14hF for an MLP exit (6hF
    forward, dM / dW_down / dW_gate|up 8hF backward: du is not needed, its
    only consumer dg_a is formed from the dW GEMM's accumulators, DESIGN.md
    §3 A28) and +18hF for a Layer exit (du feeds the attention
    block's gradient).  Layer exits add
    the attention projections, 6 (2h^2 + 2h hkv), and the causal attention
    core, 6h(T+1)/... = 2h(T+1) forward + 4h(T+1) backward (dV, dP, dQ, dK;
    the recomputed S and dP are not counted)."""
    h, V, F = cfg.hidden, cfg.vocab, cfg.ffn
    per = (4 if cfg.arch == "embedding" else 6) * h * V
    if cfg.arch == "mlp":
        per += 14 * h * F
    if cfg.arch == "layer":
        per += 18 * h * F
    if cfg.arch == "layer":
        hkv = 128 * (cfg.n_kv_heads or cfg.n_heads)
        per += 12 * h * h + 12 * h * hkv + 6 * h * (cfg.seq_len + 1)
    return per * n * cfg.exits


def attn_kw(cfg):
    """make_config / HeadSpec keywords of a Layer exit's attention geometry."""
    if cfg.arch != "layer":
        return {}
    return dict(n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads,
                seq_len=cfg.seq_len)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class OracleSample:
    """Bounded sample of the workload for the fp64 oracle: the config's exits
    at full h, V, F on n_sub tokens, each exit with its own seeded hidden
    states.  The exits share ONE seeded parameter draw (widened to fp64 once:
    7.7 GB at the 70B shape; drawing a set takes ~10 s on the host), which
    does not change the oracle's work: its time does not depend on the
    values.  Timing covers only oracle.exit_loss_and_grads (forward, CE and
    backward of an exit)."""

    def __init__(self, cfg, n_sub, seed):
        import numpy as np
        import eesynth as S
        from eesynth import to_f64
        self.cfg, self.n_sub = cfg, n_sub
        one = S.Cfg(name=cfg.name, hidden=cfg.hidden, vocab=cfg.vocab, ffn=cfg.ffn,
                    arch=cfg.arch, tokens=n_sub, layers=cfg.layers, after=list(cfg.after),
                    init=cfg.init, seed=cfg.seed, n_heads=cfg.n_heads,
                    n_kv_heads=cfg.n_kv_heads,
                    seq_len=min(cfg.seq_len, n_sub) if cfg.arch == "layer" else 0)
        self.x = [to_f64(t) for t in S.hidden_states(one, n_sub, seed=seed)]
        self.y = S.targets(one, n_sub, seed=seed).numpy().astype(np.int64)
        one.after = one.after[:1]
        one.exits = 1
        p = S.head_params(one, seed=seed)[0]
        self.params = {k: to_f64(p.pop(k)) for k in list(p)}

    def run(self, exits=None):
        """Seconds of oracle compute over `exits` (indices; default all)."""
        import eesynth as S
        from oracle import ee_oracle as O
        at = None
        if self.cfg.arch == "layer":     # the sample is one sequence of n_sub tokens
            at = dict(S.attn_geometry(self.cfg), seq_len=self.n_sub)
        total = 0.0
        for i in (range(self.cfg.exits) if exits is None else exits):
            t0 = time.perf_counter()
            O.exit_loss_and_grads(self.cfg.arch, self.params, self.x[i], self.y, 1.0, 1e-5,
                                  attn=at)
            total += time.perf_counter() - t0
        return total


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count()])
    except Exception:
        return os.cpu_count()


def cpu_baseline(cfg, args):
    """The fp64 oracle on this host's cores: all exits on n_sub tokens with
    every BLAS thread, and one exit with one thread (threadpoolctl)."""
    smp = OracleSample(cfg, args.cpu_tokens, seed=cfg.seed)
    t_all = smp.run()
    cores = oracle_threads()
    out = {"value": args.cpu_tokens / t_all, "unit": "tokens/s", "cores": cores,
           "kind": "oracle", "cpu_model": cpu_model(), "nproc": os.cpu_count(),
           "sample": f"fp64 oracle (oracle/ee_oracle.py as it stands), all {cfg.exits} exits of "
                     f"{cfg.name} on {args.cpu_tokens} tokens at full h/V/F (own hidden states, "
                     f"one shared parameter draw); {t_all:.2f} s with {cores} BLAS threads; "
                     f"Adam not included",
           "seconds": t_all}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t1 = smp.run(exits=[0])
        out["one_core"] = {"value": args.cpu_tokens / (t1 * cfg.exits), "unit": "tokens/s",
                           "cores": 1, "seconds_one_exit": t1,
                           "sample": f"exit 1 of {cfg.exits} on {args.cpu_tokens} tokens, one "
                                     f"BLAS thread; value = tokens / (t x {cfg.exits} exits)"}
    except Exception as ex:
        out["one_core"] = {"value": None, "error": repr(ex)}
    return out


def run_reference(args, cfg, rank, world):
    """--impl reference: the fp64 oracle as it stands on the host cores, rank 0
    only (other ranks exit 0).  Bounded so the driver's --steps K --warmup W
    run ends in minutes: step k runs ONE exit, exit k mod E, on n_sub =
    --ref-tokens tokens at full h/V/F, and ms_per_step is that step's
    measured time.  value = tokens/s of the whole E-exit step at that rate =
    n_sub / (E x mean step time); exit_tokens_per_s = n_sub / mean step time."""
    if rank != 0:
        return
    n_sub = args.ref_tokens
    smp = OracleSample(cfg, n_sub, seed=cfg.seed)
    times = []
    for i in range(args.warmup + args.steps):
        t = smp.run(exits=[i % cfg.exits])
        if i >= args.warmup:
            times.append(t)
    t_step = statistics.mean(times)
    value = n_sub / (t_step * cfg.exits)
    cores = oracle_threads()
    sample = (f"fp64 oracle (oracle/ee_oracle.py as it stands); each step one exit of "
              f"{cfg.exits} (rotating) of {cfg.name} on {n_sub} tokens at full h/V/F; value = "
              f"tokens / (E x step time); one shared parameter draw; Adam not included")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.scaling == "strong" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, 1, args),
            "exit_tokens_per_s": n_sub / t_step,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores,
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
                             "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def vp_comm_desc(args, vp, world):
    if getattr(args, "lib_comm", False):
        return {"dp_comm": "ee_tune_step(comm): the in-library communicator -- gradient rows "
                           "stored to their owners in the weight-gradient epilogues, owner-side "
                           "rank-ordered sums, NVLink gather of the reduced rows, rank-ordered "
                           "small reductions, device barriers (no NCCL on the step); Adam per rank"}
    if getattr(args, "dp_fused", False):
        base = "gloo" if getattr(args, "shared_gpu", False) else "NCCL"
        return {"dp_comm": "gradient reduce-scatter fused into the weight-gradient GEMM epilogues "
                           "(rows stored into their owners' arenas over CUDA-IPC peer memory), "
                           "sharded Adam storing the new operands into every rank (ZeRO-1), "
                           f"peer barriers; valid count and losses: {base}"}
    if not vp and world > 1:
        base = "gloo" if getattr(args, "shared_gpu", False) else "NCCL"
        return {"dp_comm": f"{base} all-reduce of fp32 gradients (async, overlapped) + Adam "
                           "per rank"}
    if not vp or world == 1:
        return {}
    base = "gloo" if getattr(args, "shared_gpu", False) else "NCCL"
    if getattr(args, "vp_comm", "nccl") == "fused":
        if getattr(args, "vp_zero", False):
            return {"vp_comm": "z all-gather (a4) and dz reduce-scatter (a8) fused into the "
                               "kernels, exit-body gradient rows scattered to their owners "
                               "(a11/a12 epilogues) + sharded Adam storing the body operands "
                               f"into every rank, over CUDA-IPC peer memory; CE stats: {base}"}
        return {"vp_comm": "z all-gather (a4) and dz reduce-scatter (a8) fused into the kernels "
                           f"over CUDA-IPC peer memory + peer barriers; CE stats, body grads: {base}"}
    return {"vp_comm": f"{base} all-gather / reduce-scatter"}


def tokens_per_rank(cfg, world, args):
    """Strong scaling (default; always for vp): the config's global tokens
    split over the ranks.  Weak scaling: the config's tokens on every rank."""
    if args.parallel == "vp" or args.scaling == "strong":
        if cfg.tokens % world:
            raise SystemExit(f"{cfg.tokens} tokens do not split over {world} ranks")
        return cfg.tokens // world
    return cfg.tokens


DS_LABEL = {"recompute": "recompute (a second S GEMM forms dS; no [tokens x vocab] matrix in HBM)",
            "stored_p": "stored fp16 P~ [tokens x vocab] in HBM (A24 ablation)"}


def workload_config(cfg, world, args):
    vp = args.parallel == "vp"
    tok = tokens_per_rank(cfg, world, args)
    global_tokens = cfg.tokens if (vp or args.scaling == "strong") else cfg.tokens * world
    return {"workload": f"{cfg.name}: h {cfg.hidden}, V {cfg.vocab}, F {cfg.ffn}, "
                        f"{cfg.exits} {cfg.arch} exits, {global_tokens} global tokens, "
                        f"{tok} tokens/GPU, {cfg.init} init, "
                        + (f"W_out vocab-parallel over {world}" if vp else "W_out unsharded"),
            "global_batch": max(1, global_tokens // 2048), "seq_len": 2048,
            "tokens_per_gpu": tok, "exits": cfg.exits,
            "parallelism": f"vp{world}" if vp else f"dp{world}",
            "ds": DS_LABEL[args.ds_mode],
            "collectives": ("none (one rank)" if world == 1 else
                            "gloo, ranks sharing one GPU (test mode)" if getattr(args, "shared_gpu", False)
                            else "NCCL (torch.distributed) for the small ones"),
            **vp_comm_desc(args, vp, world),
            "l2": "inputs larger than L2 (hidden states + exit weights per step >> 126 MB)",
            "optimizer": "Adam (P:374-375), included in the step",
            "update_schedule": ("per exit: W_out shard Adam + sharded exit-body Adam (ZeRO-1; "
                                "P:261)" if getattr(args, "vp_zero", False) else
                                "per exit, Adam fused into the weight-gradient epilogues "
                                "(P:261)" if getattr(args, "fused_adam", False) else
                                "per exit, each exit's Adam on a side stream overlapping the "
                                "next exit (P:261)" if getattr(args, "overlapped", False) else
                                "per exit, shared gradient buffers (P:261)"
                                if getattr(args, "per_exit", False) else
                                "per exit: tune with the gradient rows stored to their owners, "
                                "peer barrier, sharded Adam (ZeRO-1; P:261)"
                                if getattr(args, "dp_fused", False) else
                                "all exits in one ee_tune_step(comm) call, then Adam"
                                if getattr(args, "lib_comm", False) else "all exits, then Adam")}


LLAMA2 = {4096: (32, 32), 5120: (40, 40), 8192: (64, 8)}   # hidden -> (heads, kv heads) [ext]


def bench_backbone(ee, torch, cfg, args, dev):
    """Frozen backbone partial forward (ee_backbone_forward) over
    args.backbone_layers Llama-2 layers at the config's shape, on the same
    token batch; CUDA-event timed (3 warm-ups)."""
    h, F, T = cfg.hidden, cfg.ffn, 2048
    nh, nkv = LLAMA2[h]
    n = cfg.tokens
    L = args.backbone_layers
    g = torch.Generator(device=dev).manual_seed(11)

    def r(*shape):
        return (torch.randn(*shape, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    layers = [{"g_att": torch.ones(h, device=dev), "w_q": r(h, h), "w_k": r(128 * nkv, h),
               "w_v": r(128 * nkv, h), "w_o": r(h, h), "g_mlp": torch.ones(h, device=dev),
               "w_gate": r(F, h), "w_up": r(F, h), "w_down": r(h, F)} for _ in range(L)]
    x0 = torch.randn(n, h, generator=g, device=dev).to(torch.bfloat16)
    bc = ee.make_backbone_config(h, nh, nkv, F, T)
    ws = torch.empty(ee.ee_backbone_workspace_size(bc, n), dtype=torch.uint8, device=dev)
    out = [torch.empty(n, h, dtype=torch.bfloat16, device=dev)]
    for _ in range(3):
        ee.ee_backbone_forward(bc, layers, x0, [L], out, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee.ee_profile_start()
    e0.record()
    steps = max(1, args.steps // 2)
    for _ in range(steps):
        ee.ee_backbone_forward(bc, layers, x0, [L], out, ws)
    e1.record()
    torch.cuda.synchronize()
    prof = ee.ee_profile_stop()
    ms = e0.elapsed_time(e1) / steps
    flops = sum(p[3] for p in prof) / steps
    peaks = load_peaks()
    att = sum(p[1] for p in prof if p[0] == "bb_attention") / steps
    return {"layers": L, "shape": f"h {h}, heads {nh}/{nkv} kv, F {F}, seq 2048",
            "tokens": n, "ms": ms, "tokens_per_s": n / (ms / 1e3),
            "tflops": flops / (ms / 1e3) / 1e12,
            "pct_burst_peak": flops / (ms / 1e3) / 1e12 / peaks["bf16_tflops"],
            "attention_share": att / ms}


def run_pipeline(args, cfg, world, rank, local, torch, dist, ee, S):
    """--parallel pp: one EE-Tuning iteration of the paper's customised
    pipeline schedule "with forward communication only" (Fig. 3)
    including the frozen backbone's partial forward: the backbone's
    layers 1..max(exit layer) are split into `world` contiguous stages; per
    microbatch, stage s receives the activation from s-1, runs its layers
    (ee_backbone_forward, keeping the hidden states at its exits), sends the
    result to s+1 and then runs forward, loss and backward of its own exits
    (ee_tune_step, gradients accumulated over the microbatches, global valid
    count); Adam on its exits after the last microbatch.  Nothing is sent
    backward and no backbone activation is kept.  Synthetic backbone weights
    (N(0, 0.02^2), Llama-2 shapes), random exit init.  value = global tokens
    per second of the whole iteration (backbone + exits)."""
    from paper_2402_00518_b200.parallel import pipeline_forward_only_step
    ndev = torch.cuda.device_count()
    shared_gpu = world > ndev
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    multi = world > 1
    if multi:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    h, F, T = cfg.hidden, cfg.ffn, 2048
    nh, nkv = LLAMA2[h]
    Ltot = max(cfg.after)
    per = -(-Ltot // world)
    lb, le = min(Ltot, rank * per), min(Ltot, (rank + 1) * per)
    mine = [i for i, a in enumerate(cfg.after) if lb < a <= le]
    N = cfg.tokens
    if args.micro <= 0:
        args.micro = 1 if world == 1 else min(N // T, 2 * world)
    if N % (args.micro * T):
        raise SystemExit(f"{N} tokens do not split into {args.micro} microbatches of whole "
                         f"{T}-token sequences")
    mb = N // args.micro
    g = torch.Generator(device=dev).manual_seed(1000 + rank)

    def r(*shape):
        return (torch.randn(*shape, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    layers = [{"g_att": 1 + 0.1 * torch.randn(h, generator=g, device=dev),
               "w_q": r(h, h), "w_k": r(128 * nkv, h), "w_v": r(128 * nkv, h), "w_o": r(h, h),
               "g_mlp": 1 + 0.1 * torch.randn(h, generator=g, device=dev),
               "w_gate": r(F, h), "w_up": r(F, h), "w_down": r(h, F)} for _ in range(le - lb)]
    bc = ee.make_backbone_config(h, nh, nkv, F, T)
    wsb = torch.zeros(ee.ee_backbone_workspace_size(bc, mb), dtype=torch.uint8, device=dev)
    heads = None
    if mine:
        heads = ee.ExitHeads(ee.HeadSpec(h, cfg.vocab, F, len(mine), cfg.arch,
                                         ds_mode=args.ds_mode), mb, device=dev)
        heads.init("random", seed=7 + rank)
    x0 = S.hidden_states(S.Cfg(name=cfg.name, hidden=h, vocab=cfg.vocab, ffn=F, arch=cfg.arch,
                               tokens=N, layers=1, after=[1], init="random", seed=cfg.seed),
                         N, seed=cfg.seed, device=dev)[0] if rank == 0 else None
    targets = S.targets(cfg, N, seed=cfg.seed, device=dev)
    W = torch.zeros(1, dtype=torch.int64, device=dev)
    ee.ee_count_valid(targets, cfg.vocab, W, wsb)           # every stage sees every target
    outs_idx = sorted({cfg.after[i] - lb for i in mine} | {le - lb})
    bufs = {j: torch.empty(mb, h, dtype=torch.bfloat16, device=dev) for j in outs_idx}
    recv_buf = torch.empty(mb, h, dtype=torch.bfloat16, device=dev)
    total_iters = 40000

    def send(m, t):
        if shared_gpu:
            return dist.isend(t.cpu(), dst=rank + 1)
        return dist.isend(t, dst=rank + 1)

    def recv(m):
        if shared_gpu:
            c = torch.empty(mb, h, dtype=torch.bfloat16)
            dist.recv(c, src=rank - 1)
            recv_buf.copy_(c)
        else:
            dist.recv(recv_buf, src=rank - 1)
        return recv_buf

    def fwd(m, x_in):
        x = x0[m * mb:(m + 1) * mb] if x_in is None else x_in
        ee.ee_backbone_forward(bc, layers, x, outs_idx, [bufs[j] for j in outs_idx], wsb)
        return bufs[le - lb]

    def exits(m):
        if heads is None:
            return
        heads.step([bufs[cfg.after[i] - lb] for i in mine], targets[m * mb:(m + 1) * mb],
                   accumulate=m > 0, valid_count=W)

    def step(it):
        pipeline_forward_only_step(rank, world, args.micro, fwd, exits,
                                   send if rank + 1 < world else None,
                                   recv if rank > 0 else None,
                                   (lambda: heads.adam(ee.ee_lr_at(min(it + 1, total_iters),
                                                                   total_iters)))
                                   if heads is not None else None)

    def sync():
        torch.cuda.synchronize()
        if multi:
            dist.barrier()

    sync()
    for it in range(args.warmup):
        step(it)
    sync()
    sampler = ClockSampler(local % ndev)
    sampler.start()
    time.sleep(0.3)
    l0 = ee.ee_launch_count()
    ee.ee_profile_start()
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(args.steps):
        step(args.warmup + it)
    e1.record()
    sync()
    prof = ee.ee_profile_stop()
    launches = ee.ee_launch_count() - l0
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if multi:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    fl = torch.tensor([sum(p[3] for p in prof) / args.steps], dtype=torch.float64, device=dev)
    bb = torch.tensor([sum(p[1] for p in prof if p[0].startswith("bb_")) / args.steps],
                      dtype=torch.float64, device=dev)
    if multi:
        dist.all_reduce(fl)
    status = heads.status() if heads is not None else (0, -1)
    if rank == 0:
        peaks = load_peaks()
        tf = fl.item() / (ms / 1e3) / 1e12 / world
        line = {"metric": METRIC, "value": N / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (seeded backbone weights and inputs)",
                "config": {"workload": f"{cfg.name}: frozen backbone layers 1..{Ltot} (h {h}, "
                                       f"heads {nh}/{nkv} kv, F {F}) + {cfg.exits} {cfg.arch} "
                                       f"exits at layers {cfg.after}, {N} tokens per step "
                                       f"({args.micro} microbatches of {mb})",
                           "global_batch": N // T, "seq_len": T,
                           "parallelism": f"pp{world} (forward-communication-only schedule, "
                                          "P:294-303)",
                           "stage_layers": f"{per} layers per stage",
                           "ds": DS_LABEL[args.ds_mode],
                           "l2": "inputs larger than L2",
                           "optimizer": "Adam on each stage's exits after the last microbatch"},
                "pct_peak": {"algorithmic_tflops_per_gpu": tf,
                             "of_burst": tf / peaks["bf16_tflops"],
                             "step_flops_alg": fl.item()},
                "backbone_ms_rank0": bb.item(),
                "gpu_launches": launches, "clocks": clocks, "status": status}
        print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_ranks(args):
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1.  Under torchrun, --gpus
    must equal WORLD_SIZE (a mismatch would time the wrong job)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
            print("[bench] launching: " + " ".join(cmd), file=sys.stderr, flush=True)
            sys.exit(subprocess.run(cmd).returncode)
        return
    if int(ws) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; pass --gpus {ws}")


def rank_evidence(torch, dev, rank):
    p = torch.cuda.get_device_properties(dev)
    return {"rank": rank, "device": dev.index, "name": p.name,
            "pci_bus_id": getattr(p, "pci_bus_id", None),
            "uuid": str(getattr(p, "uuid", "")), "host": os.uname().nodename,
            "visible": os.environ.get("CUDA_VISIBLE_DEVICES")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="70b_dp")
    ap.add_argument("--tokens", type=int, default=0,
                    help="override the config's tokens (global under strong scaling)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="dp: strong = the config's global tokens split over the ranks "
                         "(default); weak = the config's tokens on every rank")
    ap.add_argument("--ds-mode", default="recompute", choices=["recompute", "stored_p"],
                    help="a7: recompute S for dS (default, north_star) or the stored-P~ "
                         "ablation (A24)")
    ap.add_argument("--no-ds-ablation", action="store_true",
                    help="N=1: skip timing the other ds_mode beside the headline")
    ap.add_argument("--cpu-tokens", type=int, default=64,
                    help="token sample of the fp64 oracle in cpu_baseline (all exits)")
    ap.add_argument("--ref-tokens", type=int, default=32,
                    help="--impl reference: tokens of the one exit each step runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="ncu/profiling run: no extras")
    ap.add_argument("--backbone-layers", type=int, default=0,
                    help="also time the frozen backbone partial forward (NEXT #3, P:260) over "
                         "this many Llama-2 layers of the config's shape (70b: 20 = 1/4 depth)")
    ap.add_argument("--grad-buffers", type=int, default=-1,
                    help="non-fused paths, k < exits: exits share k gradient buffers and are "
                         "updated one by one (P:261); default 2 when the config has > 4 exits")
    ap.add_argument("--dp-comm", default="fused", choices=["fused", "nccl", "plain", "lib"],
                    help="dp: fused = gradient reduce-scatter in the weight-gradient GEMM "
                         "epilogues + sharded Adam storing the operands to every rank (CUDA-IPC "
                         "peer memory, ZeRO-1; used at N=1 too); nccl = NCCL all-reduce + full "
                         "Adam per rank; plain = N=1 only: ExitHeads step + Adam (no DP machinery); "
                         "lib = one ee_tune_step(comm) call per step (the in-library DP "
                         "communicator: all-reduced gradients on every rank) + Adam per rank")
    ap.add_argument("--overlap", action="store_true",
                    help="plain N=1: exit-by-exit step with each exit's Adam on a side stream")
    ap.add_argument("--fused-adam", action="store_true",
                    help="plain N=1: Adam fused into the weight-gradient epilogues "
                         "(ee_tune_step_adam)")
    ap.add_argument("--vp-replicated-body", action="store_true",
                    help="vp fused: all-reduce the exit body's gradients and update it on "
                         "every rank instead of the sharded (ZeRO-1) body update")
    ap.add_argument("--vp-comm", default="fused", choices=["fused", "nccl"],
                    help="vp: fused = z all-gather / dz reduce-scatter inside the a4 / a8 "
                         "kernels over CUDA-IPC peer memory; nccl = NCCL collectives")
    ap.add_argument("--parallel", default="dp", choices=["dp", "vp", "pp"],
                    help="dp = data parallel over tokens; vp = W_out vocab-parallel with the "
                         "distributed softmax-CE (configs[3]: --config 70b --parallel vp); pp = "
                         "the paper's forward-communication-only pipeline with the frozen "
                         "backbone's partial forward (P:294-303, P:260; e.g. --config 13b_q)")
    ap.add_argument("--micro", type=int, default=0,
                    help="pp: microbatches per step (whole 2048-token sequences each); 0 = one "
                         "per step on one stage (larger GEMMs), 2 x stages otherwise (bubble)")
    args = ap.parse_args()
    launch_ranks(args)

    import torch
    import torch.distributed as dist
    import eesynth as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = S.get_cfg(args.config)
    if args.tokens:
        cfg.tokens = args.tokens
    args.warmup = max(args.warmup, 3 if not args.quick else args.warmup)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import paper_2402_00518_b200 as ee
    ee.load()
    if args.parallel == "pp":
        run_pipeline(args, cfg, world, rank, local, torch, dist, ee, S)
        return
    ndev = torch.cuda.device_count()
    shared_gpu = world > ndev            # test mode: several ranks on one GPU (gloo)
    args.shared_gpu = shared_gpu
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")           # per-rank init evidence (stderr)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    multi = world > 1
    ev = rank_evidence(torch, dev, rank)
    ranks = [ev]
    if multi:
        ranks = [None] * world
        dist.all_gather_object(ranks, ev)
    print(f"[bench] rank {rank}/{world}: {ev}", file=sys.stderr, flush=True)
    vp = args.parallel == "vp"
    dp = world > 1 and not vp
    n = tokens_per_rank(cfg, world, args)               # tokens of this rank's exit bodies
    n_all = cfg.tokens if vp else n
    E = cfg.exits
    from paper_2402_00518_b200.parallel import (GpuPhases, LocalComm, PeerBuffers,
                                                ShardedDPHeads, ShardedVPHeads, TorchComm,
                                                data_parallel_step, vocab_parallel_step,
                                                vocab_parallel_step_fused, vocab_shard)
    vb, ve = vocab_shard(cfg.vocab, world, rank) if vp else (0, cfg.vocab)
    spec_kw = dict(ds_mode=args.ds_mode, **attn_kw(cfg))

    # ---- parameter store, Copy init from a synthetic backbone
    if args.dp_comm == "plain" and multi:
        raise SystemExit("--dp-comm plain is the one-GPU path")
    gbuf = args.grad_buffers if args.grad_buffers >= 0 else (2 if E > 4 else 0)
    if vp or args.dp_comm == "lib":
        gbuf = 0
    dp_fused = not vp and args.dp_comm == "fused"
    heads = None
    peer_map = None
    if dp_fused:     # gradient reduce-scatter in the GEMM epilogues + sharded Adam (ZeRO-1)
        heads = ShardedDPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                           **spec_kw), n, rank, world, device=dev)
        err = None
        try:
            if world > 1:
                heads.connect_ipc()
                peer_map = {"kind": "CUDA IPC", "opened_peer_mappings": len(heads._opened)}
            else:
                heads.connect_local([heads])
                peer_map = {"kind": "local (one rank)"}
        except Exception as e:       # agree on the fallback on every rank
            err = e
        ok = torch.tensor([0 if err else 1], device=dev)
        if multi:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not ok.item():
            print(f"[bench] fused DP unavailable ({err}); using NCCL all-reduce", file=sys.stderr)
            heads.close()
            heads, dp_fused = None, False
            torch.cuda.empty_cache()
    args.dp_fused = dp_fused
    # VP with the fused collectives: the replicated exit body updated ZeRO-1 style
    vp_zero = vp and args.vp_comm == "fused" and not args.vp_replicated_body
    if vp_zero:
        heads = ShardedVPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                           **spec_kw), n_all, rank, world, device=dev)
        torch.cuda.synchronize()
        if world > 1:
            heads.connect_ipc()
        else:
            heads.connect_local([heads])
    args.vp_zero = vp_zero
    if heads is None:
        heads = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                         vocab_begin=vb, vocab_end=ve, **spec_kw), n_all,
                             device=dev, grad_buffers=gbuf if gbuf > 0 else None)
    lib_comm = None
    if not vp and args.dp_comm == "lib":
        ex = (lambda obj: (lambda out: (dist.all_gather_object(out, obj), out)[1])([None] * world)) \
            if multi else None
        lib_comm = ee.Comm(heads.cfg, "dp", world, rank, n, exchange=ex, device=dev)
        peer_map = {"kind": "ee_comm arena over CUDA IPC" if multi else "ee_comm (one rank)",
                    "arena_bytes": lib_comm.bytes}
    args.lib_comm = lib_comm is not None
    fused_adam = not multi and not vp and not dp_fused and args.fused_adam
    args.fused_adam = fused_adam
    overlapped = not multi and not vp and not dp_fused and not fused_adam and args.overlap
    args.overlapped = overlapped
    per_exit = ((not dp_fused) and (not vp_zero) and (not fused_adam) and (not overlapped)
                and lib_comm is None and heads.grad_buffers < E)
    args.per_exit = per_exit
    bb = S.backbone(cfg, device=dev)
    src = []
    for k in cfg.after:
        d = {"w_out": bb["w_out"][vb:ve]}
        if cfg.arch != "embedding":
            d["g_f"] = bb["final_norm"]
        if cfg.arch in ("mlp", "layer"):
            # MLP: the same layer's MLP; Layer: the last layer
            L = bb["layers"][k if cfg.arch == "mlp" else cfg.layers]
            d.update(g_a=L["mlp_norm"], w_gate=L["w_gate"], w_up=L["w_up"], w_down=L["w_down"])
            if cfg.arch == "layer":
                d.update({t: L[t] for t in ("g_att", "w_q", "w_k", "w_v", "w_o")})
        src.append(d)
    heads.init("copy", copy_src=src)
    torch.cuda.synchronize()
    del src, bb
    torch.cuda.empty_cache()

    if vp:
        # every rank generates the same global batch and keeps its token shard
        hidden = []
        for x in S.hidden_states(cfg, n_all, seed=cfg.seed * 100, device=dev):
            hidden.append(x[rank * n:(rank + 1) * n].contiguous())
            del x
        targets = S.targets(cfg, n_all, seed=cfg.seed * 100, device=dev)   # all tokens
        bufs = {"key": torch.zeros(n_all, dtype=torch.int64, device=dev),
                "sums": torch.zeros(n_all, 2, device=dev)}
        peer = None
        if args.vp_comm == "fused":
            peer = PeerBuffers(rank, world, n_all, cfg.hidden, device=dev)
            torch.cuda.synchronize()
            if world > 1:
                peer.connect_ipc()
            else:
                peer.connect_local([peer])
        else:
            bufs.update({"z_all": torch.zeros(n_all, cfg.hidden, dtype=torch.bfloat16, device=dev),
                         "dz_partial": torch.zeros(n_all, cfg.hidden, device=dev),
                         "dz_local": torch.zeros(n, cfg.hidden, device=dev)})
        comm = TorchComm() if world > 1 else LocalComm()
        phases = GpuPhases(ee, heads.exit_cfg if vp_zero else heads.cfg, heads.workspace)
    else:
        # strong scaling: rank r holds tokens [r n, (r+1) n) of the global batch
        # (each rank draws its own shard; seeds differ per rank)
        hidden = S.hidden_states(cfg, n, seed=cfg.seed * 100 + rank, device=dev)
        targets = S.targets(cfg, n, seed=cfg.seed * 100 + rank, device=dev)
    vc = torch.zeros(1, dtype=torch.int64, device=dev)
    job_tokens = n_all if vp else n * world
    total_iters = 40000
    one_cfg = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, cfg.arch, **spec_kw)
    all_reduce = dist.all_reduce if multi else None

    def step(it, hid=hidden, tg=targets, lr=None):
        if lr is None:
            lr = ee.ee_lr_at(min(it + 1, total_iters), total_iters)
        if fused_adam:     # one GPU: Adam fused into the weight-gradient epilogues
            heads.step_adam(hid, tg, lr)
            return
        if overlapped:     # exit by exit, each exit's Adam on a side stream overlapping the next
            heads.step_overlapped(hid, tg, lr)
            return
        if dp_fused:       # exit by exit: tune -> peer barrier -> sharded Adam
            heads.step(hid, tg, lr, all_reduce=all_reduce)
            return
        if per_exit:       # exit-by-exit update with shared gradient buffers
            W = None
            if dp:
                ee.ee_count_valid(tg, cfg.vocab, vc, heads.workspace)
                dist.all_reduce(vc)
                W = vc
            red = (lambda i: [dist.all_reduce(t, async_op=True) for t in heads.grads[i].values()]) \
                if dp else None
            heads.step_per_exit(hid, tg, lr, valid_count=W, reduce_grads=red)
            if dp:
                dist.all_reduce(heads.loss)
            return
        if vp:
            ee.ee_count_valid(tg, cfg.vocab, vc, heads.workspace)   # W over all tokens
            if vp_zero:    # body gradients to their owners, sharded Adam per exit
                heads.set_lr(lr)
                vocab_parallel_step_fused(phases, comm, peer, cfg.arch, hid, tg, heads.operand,
                                          heads.grads, heads.loss, [1.0] * E, vc, bufs,
                                          body=heads)
                return
            if peer is not None:
                vocab_parallel_step_fused(phases, comm, peer, cfg.arch, hid, tg, heads.operand,
                                          heads.grads, heads.loss, [1.0] * E, vc, bufs)
            else:
                vocab_parallel_step(phases, comm, cfg.arch, hid, tg, heads.operand, heads.grads,
                                    heads.loss, [1.0] * E, vc, bufs)
        elif lib_comm is not None:     # the whole DP step in one C-ABI call (ee_comm)
            ee.ee_tune_step(heads.cfg, hid, tg, [1.0] * E, heads.operand, heads.grads,
                            heads.loss, heads.workspace, comm=lib_comm)
        elif not dp:
            heads.step(hid, tg)
        else:
            def count_local():
                ee.ee_count_valid(tg, cfg.vocab, vc, heads.workspace)
                return vc

            def run_exit(i, W):                           # exit i on this rank's tokens
                ee.ee_tune_step(one_cfg, hid[i:i + 1], tg, [1.0], heads.operand[i:i + 1],
                                heads.grads[i:i + 1], heads.loss[i:i + 1], heads.workspace,
                                valid_count=W)

            data_parallel_step(E, count_local, run_exit, lambda i: heads.grads[i].values(),
                               heads.loss)
        heads.adam(lr)

    def sync():
        torch.cuda.synchronize()
        if multi:
            dist.barrier()

    def timed(fn, steps):
        """Device time per step of `steps` calls of fn(it): CUDA events on the
        launching stream, barrier + synchronize on both sides, max over ranks."""
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(steps):
            fn(it)
        if hasattr(heads, "join"):
            heads.join()            # the last side-stream update is inside the timed region
        e1.record()
        sync()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    sync()          # line the ranks up before the first peer barrier (its timeout is 20 s)
    for it in range(args.warmup):
        step(it)
    sync()

    # ---- timed region (device time, CUDA events on the launching stream)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = ee.ee_launch_count()
    ee.ee_profile_start()
    ms = timed(lambda it: step(args.warmup + it), args.steps)
    prof = ee.ee_profile_stop()
    launches = ee.ee_launch_count() - l0
    clocks = sampler.stop()
    code, idx = heads.status()
    it_done = args.warmup + args.steps

    # ---- the other ds_mode, timed the same way beside the headline (N = 1)
    ablation = None
    if world == 1 and not args.quick and not args.no_ds_ablation and not vp:
        other = "stored_p" if args.ds_mode == "recompute" else "recompute"
        cfgs = [getattr(heads, "cfg", None), getattr(heads, "exit_cfg", None)]
        for c in cfgs:
            if c is not None:
                c.ds_mode = ee.DS_MODE[other]
        one_cfg.ds_mode = ee.DS_MODE[other]
        step(it_done)
        sampler2 = ClockSampler(local)
        sampler2.start()
        abl_steps = min(args.steps, 5)          # bounded: a secondary number
        ms_o = timed(lambda it: step(it_done + 1 + it), abl_steps)
        cl2 = sampler2.stop()
        for c in cfgs:
            if c is not None:
                c.ds_mode = ee.DS_MODE[args.ds_mode]
        one_cfg.ds_mode = ee.DS_MODE[args.ds_mode]
        it_done += 1 + abl_steps
        ablation = {"ds": DS_LABEL[other], "value": job_tokens / (ms_o / 1e3),
                    "unit": "tokens/s", "ms_per_step": ms_o, "steps": abl_steps,
                    "pct_of_burst_peak": step_flops(cfg, n) / (ms_o / 1e3) / 1e12
                    / load_peaks()["bf16_tflops"], "sm_mhz": cl2.get("sm_mhz")}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and not args.quick:
        h_host = [h.cpu().pin_memory() for h in hidden]
        t_host = targets.cpu().pin_memory()
        loss_host = torch.empty(E, dtype=torch.float32).pin_memory()
        # two input sets without a second copy in host memory: set B feeds
        # exit i the hidden states of exit (i+1) mod E (a staging race that
        # mixed buffers or calls would change the losses)
        perm = [(i + 1) % E for i in range(E)]
        sets_host = [(h_host, t_host), ([h_host[j] for j in perm], t_host)]
        sets_dev = [(hidden, targets), ([hidden[j] for j in perm], targets)]
        streamed = not vp and not per_exit and lib_comm is None and (dp_fused or not multi)
        check = None
        if streamed:
            # correctness of the host-input path on alternating sets, lr = 0
            # (Adam with lr 0 leaves the parameters bitwise unchanged)
            def dev_step(hs, tg):
                if dp_fused:
                    heads.step(hs, tg, 0.0, all_reduce=all_reduce)
                else:
                    heads.step(hs, tg)
                return heads.loss.clone()

            def host_step(hs, tg, lr):
                if dp_fused:
                    heads.step_host(hs, tg, lr, all_reduce=all_reduce)
                elif overlapped or fused_adam:
                    heads.step_host(hs, tg, lr=lr, fused_adam=fused_adam)
                else:
                    heads.step_host(hs, tg)
                    if lr is not None:
                        heads.adam(lr)
                return heads.loss

            want = [dev_step(*sets_dev[k]) for k in range(2)]
            got = [host_step(*sets_host[r % 2], 0.0 if (dp_fused or overlapped or fused_adam)
                             else None).clone() for r in range(4)]
            sync()
            ok = all(torch.equal(got[r], want[r % 2]) for r in range(4))
            check = {"alternating_sets_bitwise_equal_device_step": ok,
                     "loss_set_a": [round(float(v), 6) for v in want[0].tolist()],
                     "loss_set_b": [round(float(v), 6) for v in want[1].tolist()]}
            if not ok:
                print(f"[bench] e2e check FAILED: {got} vs {want}", file=sys.stderr, flush=True)
        sync()

        def e2e_step(it):
            hs, tg = sets_host[it % 2]
            lr = ee.ee_lr_at(min(it_done + it + 1, total_iters), total_iters)
            if streamed:      # per-exit H2D overlapped with the previous exit's compute
                host_step(hs, tg, lr)
            else:
                hd, td = sets_dev[it % 2]
                for d_, h_ in zip(hidden, h_host):
                    d_.copy_(h_, non_blocking=True)
                targets.copy_(t_host, non_blocking=True)
                step(it_done + it, hid=hd, tg=td, lr=lr)
            loss_host.copy_(heads.loss, non_blocking=True)
        te = timed(e2e_step, args.steps)
        e2e = {"value": job_tokens / (te / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": sum(h.numel() * 2 for h in hidden) + targets.numel() * 4,
               "d2h_bytes_per_step": E * 4, "ms_per_step": te,
               "inputs": "pinned host memory, two alternating input sets",
               "api": ("ShardedDPHeads.step_host (per-exit H2D overlapped with compute)"
                       if dp_fused and streamed else
                       "ExitHeads.step_host (per-exit H2D overlapped with compute)"
                       if streamed else "H2D copies + step"),
               "check": check}
        del h_host, sets_host

    if rank != 0:
        if multi:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- per-kernel breakdown of the timed region
    peaks = load_peaks()
    kern = {}
    for name, kms, fe, fa, by in prof:
        d = kern.setdefault(name, {"launches": 0, "ms": 0.0, "flops_exec": 0.0, "flops_alg": 0.0,
                                   "bytes": 0.0})
        d["launches"] += 1
        d["ms"] += kms
        d["flops_exec"] += fe
        d["flops_alg"] += fa
        d["bytes"] += by
    step_ms_sum = sum(d["ms"] for d in kern.values())
    kernels = {}
    for name, d in sorted(kern.items(), key=lambda kv: -kv[1]["ms"]):
        e = {"launches_per_step": d["launches"] / args.steps, "ms_per_launch": d["ms"] / d["launches"],
             "share": d["ms"] / step_ms_sum if step_ms_sum else None}
        if d["flops_exec"]:
            e["tflops_exec"] = d["flops_exec"] / (d["ms"] / 1e3) / 1e12
        if d["bytes"]:
            e["gbs"] = d["bytes"] / (d["ms"] / 1e3) / 1e9
        kernels[name] = e
    gemms = {k: v for k, v in kern.items() if v["flops_alg"] > 0}
    dom = max(gemms, key=lambda k: gemms[k]["ms"]) if gemms else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    roofline = None
    if dom:
        d = gemms[dom]
        per_launch_flops = d["flops_alg"] / d["launches"]
        ach = per_launch_flops / (d["ms"] / d["launches"] / 1e3) / 1e12
        # the sustained peak for a kernel timed inside a timed region of >= 1 s
        # (the power-capped regime MEASURED_PEAKS' sustained figure was taken
        # in), the burst peak for a short one (e.g. 7b: 5 x 20 ms at max clock)
        long_region = ms * args.steps >= 1000.0
        pk = peaks["bf16_tflops_sustained"] if long_region else peaks["bf16_tflops"]
        roofline = {"bound": "tensor", "kernel": dom, "achieved": ach,
                    "peak": pk, "unit": "TFLOP/s",
                    "frac": ach / pk, "frac_of_burst": ach / peaks["bf16_tflops"],
                    "traffic": traffic,
                    "algorithmic_flops_per_launch": per_launch_flops,
                    "peak_source": peaks["source"] + (
                        ", sustained (kernel timed inside a timed region of >= 1 s)" if long_region
                        else ", burst (timed region < 1 s)")}

    F_alg = step_flops(cfg, n_all if vp else n)          # per GPU for dp, whole job for vp
    exec_tflops = sum(d["flops_exec"] for d in kern.values()) / args.steps / (ms / 1e3) / 1e12
    tflops = F_alg / (ms / 1e3) / 1e12 / (world if vp else 1)
    value = job_tokens / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if (vp or args.scaling == "strong") else "weak",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded eesynth inputs, Copy init from a synthetic backbone)",
        "config": workload_config(cfg, world, args),
        "pct_peak": {"algorithmic_tflops_per_gpu": tflops,
                     "of_burst": tflops / peaks["bf16_tflops"],
                     "of_sustained": tflops / peaks["bf16_tflops_sustained"],
                     "of_datasheet_2250": tflops / 2250.0,
                     "step_flops_alg_per_gpu": F_alg / (world if vp else 1),
                     # executed tensor work incl. the dS recompute GEMM (not credited above)
                     "executed_tflops_per_gpu": exec_tflops,
                     "executed_of_burst": exec_tflops / peaks["bf16_tflops"],
                     "peak_source": peaks["source"]},
        "roofline": roofline,
        # exit-tokens/s (comparable across exit counts) and the
        # optimizer's share, reported beside the step that includes it
        "exit_tokens_per_s": E * job_tokens / (ms / 1e3),
        "update_ms_per_step": sum(d["ms"] for k, d in kern.items() if k.startswith("a15"))
                              / args.steps,
        "ds_ablation": ablation,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "status": code,
        "ranks": ranks,
        "peer_map": peer_map,
        "loss_last_step": [round(float(v), 6) for v in heads.loss.tolist()],
        "kernels": kernels,
    }
    if args.backbone_layers > 0 and world == 1:
        line["backbone_forward"] = bench_backbone(ee, torch, cfg, args, dev)
    if world == 1 and not args.no_cpu_baseline and not args.quick:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args)
        except Exception as ex:  # never let the baseline kill the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(),
                                    "kind": "oracle", "sample": f"failed: {ex!r}"}
    print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
