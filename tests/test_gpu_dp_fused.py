"""Fused data-parallel path (include/ee.h ee_tune_step_rs /
ee_adam_update_sharded; parallel.ShardedDPHeads): the weight-gradient GEMM
epilogues store every gradient row into its owner's arena, the owner sums the
slots in rank order, runs Adam on its master/moment shard and stores the new
operand rows into every rank (ZeRO-1 without NCCL on the bulk path).

P ranks are emulated by P host threads on their own CUDA streams (the device
peer barrier really synchronises them).  After two steps every rank's bf16
operands and fp32 master rows must equal, BIT FOR BIT, those of the
all-reduce path (ee_tune_step on the token shard + rank-ordered fp32 sum of
the gradients + ee_adam_update on the full tensors), and the losses must match
the fp64 oracle (north_star tolerance).  A two-process CUDA-IPC run covers
connect_ipc.
"""

import os
import threading

import numpy as np
import pytest
import torch

import eesynth as S
from harness import LOSS_RTOL, oracle_exit
from test_gpu_vp_fused import StreamThreadComm

pytestmark = pytest.mark.gpu


def _cfg(arch, seed, exits=3):
    if arch == "layer":     # 4 sequences of 128 tokens (whole sequences per rank)
        c = S.get_cfg("tiny_layer", seed=seed)
        c.tokens = 512
        return c
    return S.Cfg(name="small", hidden=128, vocab=1000, ffn=256 if arch == "mlp" else 0,
                 arch=arch, tokens=256, layers=exits, after=list(range(1, exits + 1)),
                 init="random", seed=seed)


def _attn(cfg):
    if cfg.arch != "layer":
        return {}
    return dict(n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads,
                seq_len=cfg.seq_len)


def _copy_src(params):
    return [{k: v.cuda().float().contiguous() for k, v in p.items()} for p in params]


def run_threads(ee, cfg, P, hidden, targets, params, fused, steps=2, n_arenas=2):
    from paper_2402_00518_b200.parallel import ShardedDPHeads
    N, E = targets.numel(), cfg.exits
    nl = N // P
    spec = ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch, **_attn(cfg))
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": [None] * P}
    heads = [ShardedDPHeads(spec, nl, r, P, n_arenas=n_arenas) for r in range(P)] if fused \
        else None
    if fused:
        for h in heads:
            h.connect_local(heads)
    torch.cuda.synchronize()
    out, errors = [None] * P, []

    def rank_fn(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = StreamThreadComm(shared, r, st)
                hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
                tg = targets[r * nl:(r + 1) * nl].cuda().contiguous()
                losses = []
                if fused:
                    hd = heads[r]
                    hd.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
                    for it in range(steps):
                        losses.append(hd.step(hid, tg, 1e-3 * (it + 1),
                                              all_reduce=lambda t: comm.all_reduce(t)).cpu())
                    master = [{k: v.cpu() for k, v in d.items()} for d in hd.master]
                    operand = [{k: v.cpu() for k, v in d.items()} for d in hd.operand]
                    layout = hd.layout
                    ws = hd.workspace
                else:
                    hd = ee.ExitHeads(spec, nl)
                    hd.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
                    W = torch.zeros(1, dtype=torch.int64, device="cuda")
                    for it in range(steps):
                        ee.ee_count_valid(tg, cfg.vocab, W, hd.workspace)
                        comm.all_reduce(W)
                        hd.step(hid, tg, valid_count=W)
                        for g in hd.grads:
                            for t in g.values():
                                comm.all_reduce(t)
                        hd.adam(1e-3 * (it + 1))
                        comm.all_reduce(hd.loss)
                        losses.append(hd.loss.cpu())
                    master = [{k: v.cpu() for k, v in d.items()} for d in hd.master]
                    operand = [{k: v.cpu() for k, v in d.items()} for d in hd.operand]
                    layout = None
                    ws = hd.workspace
                st.synchronize()
                out[r] = (losses, master, operand, layout, ee.ee_get_status(ws, stream=st))
        except Exception as e:  # surface thread failures
            errors.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errors:
        raise errors[0]
    return out


def _warm(ee, cfg, hidden, targets, params):
    """One world-1 fused step first.  CUDA loads kernels lazily, and loading
    a kernel waits for the context's running kernels: with all emulated ranks
    in ONE context, a rank's first launch of a kernel would wait for another
    rank's spinning peer barrier, which waits for that first rank (deadlock
    until the barrier's timeout).  One process per GPU has no such cycle."""
    run_threads(ee, cfg, 1, hidden, targets, params, fused=True, steps=1)


@pytest.mark.parametrize("arch,P,n_arenas", [("mlp", 2, 2), ("mlp", 4, 2), ("norm", 4, 2),
                                             ("embedding", 2, 2), ("mlp", 1, 2), ("mlp", 3, 1),
                                             ("mlp", 8, 2), ("layer", 2, 2), ("layer", 4, 2)])
def test_fused_dp_bitwise_equals_allreduce_path(gpu_lib, arch, P, n_arenas):
    ee = gpu_lib
    cfg = _cfg(arch, 51)
    N = 240 if P == 3 else (cfg.tokens if arch == "layer" else 256)
    hidden = S.hidden_states(cfg, N)
    targets = S.targets(cfg, N)
    params = S.head_params(cfg)
    ref = run_threads(ee, cfg, P, hidden, targets, params, fused=False)
    _warm(ee, cfg, hidden, targets, params)
    fus = run_threads(ee, cfg, P, hidden, targets, params, fused=True, n_arenas=n_arenas)
    for r in range(P):
        assert fus[r][4] == (0, -1), fus[r][4]
        for it in range(2):
            assert torch.equal(fus[r][0][it], ref[r][0][it]), (r, it)
        for i in range(cfg.exits):
            for k, t in ref[r][2][i].items():            # full operands on every rank
                assert torch.equal(fus[r][2][i][k], t), (r, i, k)
            for k, full in ref[r][1][i].items():         # master rows of this rank's shard
                b, rows = fus[r][3][k][0], fus[r][3][k][1]
                want = full.reshape(-1, full.shape[-1])[b:b + rows]
                assert torch.equal(fus[r][1][i][k], want), (r, i, k)
    # first-step losses against the fp64 oracle (parameters = the Copy source)
    for i in range(cfg.exits):
        res = oracle_exit(arch, params[i], hidden[i], targets, 1.0, attn=S.attn_geometry(cfg))
        assert abs(fus[0][0][0][i].item() - res.loss) / res.loss <= LOSS_RTOL


def test_dp_shard_layout_partitions_rows(gpu_lib):
    """Shards tile each tensor's rows exactly once; arena blocks are disjoint
    and sized P x rows x C."""
    ee = gpu_lib
    for P in (1, 2, 3, 8):
        c = ee.make_config(128, 1000, 256, 1, "mlp")
        shapes = ee.tensor_shapes(128, 1000, 256, "mlp")
        for k, sh in shapes.items():
            R = 1 if len(sh) == 1 else sh[0]
            C = sh[-1]
            covered = []
            for q in range(P):
                b, rows, off, total = ee.ee_dp_shard_layout(c, P, q, k)
                covered += list(range(b, b + rows))
                assert off + P * rows * C <= total
            assert covered == list(range(R)), (P, k)


# ---------------------------------------------------------------------------
# two processes, one GPU, CUDA IPC
# ---------------------------------------------------------------------------

def _ipc_worker(rank, world, port, path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2402_00518_b200 as ee
    from paper_2402_00518_b200.parallel import ShardedDPHeads
    ee.load()
    cfg = _cfg("mlp", 61, exits=2)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    nl = 256 // world
    hd = ShardedDPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch), nl,
                        rank, world)
    torch.cuda.synchronize()
    hd.connect_ipc()
    hd.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)

    def ar(t):
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)

    hid = [x[rank * nl:(rank + 1) * nl].cuda().contiguous() for x in hidden]
    tg = targets[rank * nl:(rank + 1) * nl].cuda().contiguous()
    losses = [hd.step(hid, tg, 1e-3 * (it + 1), all_reduce=ar).cpu() for it in range(2)]
    torch.cuda.synchronize()
    st = ee.ee_get_status(hd.workspace)
    dist.barrier()
    ops = [{k: v.cpu() for k, v in d.items()} for d in hd.operand]
    hd.close()
    torch.save({"loss": losses, "operand": ops, "status": st}, f"{path}.{rank}")
    dist.destroy_process_group()


def test_fused_dp_two_processes_cuda_ipc(gpu_lib, tmp_path):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "out")
    mp.start_processes(_ipc_worker, args=(2, port, path), nprocs=2, join=True,
                       start_method="spawn")
    outs = [torch.load(f"{path}.{r}") for r in range(2)]
    cfg = _cfg("mlp", 61, exits=2)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    ref = run_threads(gpu_lib, cfg, 2, hidden, targets, params, fused=False)
    for r, o in enumerate(outs):
        assert o["status"] == (0, -1)
        for it in range(2):
            assert torch.equal(o["loss"][it], ref[r][0][it].cpu())
        for i in range(cfg.exits):
            for k, t in ref[r][2][i].items():
                assert torch.equal(o["operand"][i][k], t), (r, i, k)
    for i in range(cfg.exits):
        res = oracle_exit("mlp", params[i], hidden[i], targets, 1.0)
        assert abs(outs[0]["loss"][0][i].item() - res.loss) / res.loss <= LOSS_RTOL


def test_fused_dp_confidence_weighting_bitwise(gpu_lib):
    """Dynamic token weights under the fused DP path: ranks run
    EE_WEIGHT_CONFIDENCE_SUM into the arenas, the weight sums are all-reduced,
    the sharded Adam divides by them (grad_divisor) and the losses are divided
    with ee_normalize_exit(grads=NULL) -- bitwise the all-reduce path
    (rank-ordered sums, ee_normalize_exit on full gradients, Adam)."""
    ee = gpu_lib
    from paper_2402_00518_b200.parallel import ShardedDPHeads
    cfg = _cfg("mlp", 53)
    P, N, E = 2, 256, cfg.exits
    nl = N // P
    hidden = S.hidden_states(cfg, N)
    targets = S.targets(cfg, N)
    params = S.head_params(cfg)
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": [None] * P}
    heads = [ShardedDPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                        token_weighting="confidence"), nl, r, P)
             for r in range(P)]
    for h in heads:
        h.connect_local(heads)
    # world-1 confidence step first: loads the kernels this path adds (see _warm)
    w1 = ShardedDPHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                    token_weighting="confidence"), N, 0, 1)
    w1.connect_local([w1])
    w1.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
    w1.step([x.cuda() for x in hidden], targets.cuda(), 1e-3, all_reduce=lambda t: None)
    torch.cuda.synchronize()
    out, errors = [[None, None] for _ in range(P)], []

    def rank_fn(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = StreamThreadComm(shared, r, st)
                hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
                tg = targets[r * nl:(r + 1) * nl].cuda().contiguous()
                # fused
                hd = heads[r]
                hd.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
                for it in range(2):
                    hd.step(hid, tg, 1e-3 * (it + 1), all_reduce=lambda t: comm.all_reduce(t))
                out[r][0] = ([{k: v.cpu() for k, v in d.items()} for d in hd.operand],
                             hd.loss.cpu(), ee.ee_get_status(hd.workspace, stream=st))
                # all-reduce reference
                rf = ee.ExitHeads(ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, E, cfg.arch,
                                              token_weighting="confidence_sum"), nl)
                rf.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
                ecfg = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, cfg.arch,
                                      token_weighting="confidence_sum")
                ws = [torch.zeros(1, device="cuda") for _ in range(E)]
                for it in range(2):
                    rf.step(hid, tg, aux=[{"weight_sum": w} for w in ws])
                    for g in rf.grads:
                        for t in g.values():
                            comm.all_reduce(t)
                    comm.all_reduce(rf.loss)
                    for i in range(E):
                        comm.all_reduce(ws[i])
                        ee.ee_normalize_exit(ecfg, rf.grads[i], rf.loss[i:i + 1], ws[i])
                    rf.adam(1e-3 * (it + 1))
                out[r][1] = ([{k: v.cpu() for k, v in d.items()} for d in rf.operand],
                             rf.loss.cpu(), None)
                st.synchronize()
        except Exception as e:  # surface thread failures
            errors.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errors:
        raise errors[0]
    for r in range(P):
        got, ref = out[r]
        assert got[2] == (0, -1)
        assert torch.equal(got[1], ref[1]), (got[1], ref[1])
        for i in range(E):
            for k, t in ref[0][i].items():
                assert torch.equal(got[0][i][k], t), (r, i, k)


def test_sharded_step_host_equals_device_step(gpu_lib):
    """ShardedDPHeads.step_host (the bench's e2e API at every N: per-exit H2D
    on a copy stream, HostStager) gives bitwise the device step's losses and
    parameters, on alternating input sets issued back to back."""
    from paper_2402_00518_b200.parallel import ShardedDPHeads
    ee = gpu_lib
    cfg = _cfg("mlp", 31)
    spec = ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch)
    params = S.head_params(cfg)
    sets = [(S.hidden_states(cfg, 256, seed=s), S.targets(cfg, 256, seed=s)) for s in (1, 2)]
    runs = []
    for host in (False, True):
        hd = ShardedDPHeads(spec, 256, 0, 1)
        hd.connect_local([hd])
        hd.init("copy", copy_src=_copy_src(params), src_dtype=torch.float32)
        losses = []
        for it in range(6):
            hs, t = sets[it % 2]
            if host:
                hd.step_host([h.pin_memory() for h in hs], t.pin_memory(), 1e-3)
            else:
                hd.step([h.cuda() for h in hs], t.cuda(), 1e-3)
            losses.append(hd.loss.clone())
        torch.cuda.synchronize()
        runs.append((losses, [{k: v.clone() for k, v in d.items()} for d in hd.operand]))
    for a, b in zip(runs[0][0], runs[1][0]):
        assert torch.equal(a, b)
    for i in range(cfg.exits):
        for k in runs[0][1][i]:
            assert torch.equal(runs[0][1][i][k], runs[1][1][i][k]), (i, k)
