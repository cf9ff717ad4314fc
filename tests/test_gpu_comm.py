"""The in-library communicator (include/ee.h ee_comm_*): ONE ee_tune_step call
runs the whole data-parallel or vocab-parallel step (§2.2 "Support
for 3D parallelism"), with every exchange done by the library's
kernels over peer memory.

1. P ranks emulated by P host threads, each on its own CUDA stream (the
   device barriers really synchronise them), against the fp64 oracle on ALL
   tokens: the DP-summed gradient of every tensor on every rank (north_star
   bound), bitwise identical across ranks, the global loss; VP: the
   concatenated W_out shard gradients and the all-reduced body gradients.
   Dynamic token weights are normalised by the global sum_t c_t.
2. Two processes on the same GPU, arenas mapped with CUDA IPC and the handles
   exchanged over a TCPStore (no process group, no gloo, no NCCL): each rank
   calls only ee_tune_step(comm) and must match the oracle.
"""

import os
import threading

import numpy as np
import pytest
import torch

import eesynth as S
from harness import GRAD_RTOL, grad_rtol, LOSS_RTOL, attn_kwargs, oracle_exit, rel_fro

pytestmark = pytest.mark.gpu


def _cfg(arch, seed):
    if arch == "layer":     # 4 sequences of 128 tokens (whole sequences per rank)
        c = S.get_cfg("tiny_layer", seed=seed)
        c.tokens = 512
        return c
    return S.Cfg(name="small", hidden=128, vocab=1000, ffn=256 if arch == "mlp" else 0,
                 arch=arch, tokens=384, layers=2, after=[1, 2], init="random", seed=seed)


def _rank_setup(ee, cfg, mode, P, r, params, hidden, weighting):
    from paper_2402_00518_b200.parallel import vocab_shard
    N = hidden[0].shape[0]
    nl = N // P
    vb, ve = vocab_shard(cfg.vocab, P, r) if mode == "vp" else (0, cfg.vocab)
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch, 1e-5, vb, ve,
                       token_weighting=weighting, **attn_kwargs(cfg))
    prm, grd = [], []
    for p in params:
        d = {}
        for k, v in p.items():
            v = v[vb:ve] if k == "w_out" else v
            d[k] = v.cuda().float().contiguous() if k.startswith("g_") else \
                v.cuda().to(torch.bfloat16).contiguous()
        prm.append(d)
        grd.append({k: torch.full(d[k].shape, float("nan"), device="cuda") for k in d})
    ws = torch.zeros(ee.ee_workspace_size(c, N if mode == "vp" else nl), dtype=torch.uint8,
                     device="cuda")
    hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
    return c, prm, grd, ws, hid


def _run(ee, cfg, mode, P, hidden, targets, params, weights, weighting="uniform", steps=1):
    """Every rank on its own thread and stream calls ee_tune_step(comm=...)."""
    N = targets.numel()
    nl = N // P
    setups = [_rank_setup(ee, cfg, mode, P, r, params, hidden, weighting) for r in range(P)]
    comms = ee.Comm.local([s[0] for s in setups], mode, P, nl)
    out, errors = [None] * P, []

    def rank_fn(r):
        try:
            c, prm, grd, ws, hid = setups[r]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                tg = targets[r * nl:(r + 1) * nl].cuda().contiguous()
                loss = torch.full((cfg.exits,), float("nan"), device="cuda")
                for _ in range(steps):
                    ee.ee_tune_step(c, hid, tg, weights, prm, grd, loss, ws, comm=comms[r],
                                    stream=st)
                st.synchronize()
                out[r] = (loss.cpu(), [{k: v.cpu() for k, v in g.items()} for g in grd],
                          ee.ee_get_status(ws, stream=st))
        except Exception as e:  # surface thread failures
            errors.append(e)

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    torch.cuda.synchronize()
    for cm in comms:
        cm.close()
    assert not errors, errors
    return out


_warmed = set()


def _warm(ee, mode, arch, weighting="uniform"):
    """A world-1 comm step first, with the same arch and token weighting:
    CUDA loads kernels lazily and a module load waits for the context's
    running kernels, so a thread-rank's first launch of a kernel could
    otherwise wait behind another rank's spinning barrier (include/ee.h)."""
    if (mode, arch, weighting) in _warmed:
        return
    cfg = _cfg(arch, 1)
    n = 256 if arch == "layer" else 64
    hidden = S.hidden_states(cfg, n)
    _run(ee, cfg, mode, 1, hidden, S.targets(cfg, n), S.head_params(cfg), [1.0, 1.0],
         weighting=weighting)
    _warmed.add((mode, arch, weighting))


def _check_vs_oracle(cfg, mode, P, out, hidden, targets, params, weights, weighting="uniform"):
    at = S.attn_geometry(cfg)
    for r in range(P):
        assert out[r][2] == (0, -1), out[r][2]
    for i, a in enumerate(weights):
        res = oracle_exit(cfg.arch, params[i], hidden[i], targets, a, weighting=weighting,
                          attn=at)
        for r in range(P):
            L = out[r][0][i].item()
            assert abs(L - res.loss) / res.loss <= LOSS_RTOL, (r, i, L, res.loss)
            assert torch.equal(out[r][0], out[0][0])                  # same loss everywhere
        errs = {}
        for k, g in res.grads.items():
            if mode == "vp" and k == "w_out":
                got = torch.cat([out[r][1][i]["w_out"] for r in range(P)])
            else:
                got = out[0][1][i][k]
                for r in range(1, P):                                 # all-reduced: identical
                    assert torch.equal(out[r][1][i][k], got), (r, i, k)
            errs[k] = rel_fro(got.double().numpy(), g)
            assert errs[k] <= grad_rtol(cfg.arch, k), (i, k, errs[k])
        print(mode, cfg.arch, P, weighting, i, {k: f"{e:.1e}" for k, e in errs.items()})


@pytest.mark.parametrize("arch,P", [("mlp", 2), ("mlp", 4), ("norm", 3), ("embedding", 2),
                                    ("layer", 2)])
def test_dp_comm_one_call_matches_oracle(gpu_lib, arch, P):
    _warm(gpu_lib, "dp", arch)
    cfg = _cfg(arch, 60 + P)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    out = _run(gpu_lib, cfg, "dp", P, hidden, targets, params, [1.0, 0.5])
    _check_vs_oracle(cfg, "dp", P, out, hidden, targets, params, [1.0, 0.5])


def test_dp_comm_confidence_weighting_global_normaliser(gpu_lib):
    """P:326-336 / App. B.3: w_t = c_t detached, normalised by sum_t c_t over
    the tokens of ALL ranks (A17)."""
    _warm(gpu_lib, "dp", "mlp", "confidence")
    cfg = _cfg("mlp", 71)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    out = _run(gpu_lib, cfg, "dp", 2, hidden, targets, params, [1.0, 0.5],
               weighting="confidence")
    _check_vs_oracle(cfg, "dp", 2, out, hidden, targets, params, [1.0, 0.5],
                     weighting="confidence")


def test_dp_comm_repeat_calls_bitwise(gpu_lib):
    """Three calls in a row end with bitwise the result of one call: the
    arenas, the small reduction slots and the barrier epochs are reusable."""
    _warm(gpu_lib, "dp", "mlp")
    cfg = _cfg("mlp", 72)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    a = _run(gpu_lib, cfg, "dp", 2, hidden, targets, params, [1.0, 0.5], steps=1)
    b = _run(gpu_lib, cfg, "dp", 2, hidden, targets, params, [1.0, 0.5], steps=3)
    for r in range(2):
        assert torch.equal(a[r][0], b[r][0])
        for i in range(2):
            for k in a[r][1][i]:
                assert torch.equal(a[r][1][i][k], b[r][1][i][k]), (r, i, k)


@pytest.mark.parametrize("arch,P", [("mlp", 2), ("mlp", 4), ("embedding", 2), ("layer", 2)])
def test_vp_comm_one_call_matches_oracle(gpu_lib, arch, P):
    _warm(gpu_lib, "vp", arch)
    cfg = _cfg(arch, 80 + P)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    out = _run(gpu_lib, cfg, "vp", P, hidden, targets, params, [1.0, 0.5])
    _check_vs_oracle(cfg, "vp", P, out, hidden, targets, params, [1.0, 0.5])


def test_vp_comm_confidence_weighting(gpu_lib):
    _warm(gpu_lib, "vp", "mlp", "confidence")
    cfg = _cfg("mlp", 73)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    out = _run(gpu_lib, cfg, "vp", 2, hidden, targets, params, [1.0, 0.5],
               weighting="confidence")
    _check_vs_oracle(cfg, "vp", 2, out, hidden, targets, params, [1.0, 0.5],
                     weighting="confidence")


# ---------------------------------------------------------------------------
# two processes, handles over a TCPStore: nothing but ee_tune_step(comm)
# ---------------------------------------------------------------------------

def _store_worker(rank, world, port, path, mode):
    from datetime import timedelta

    import torch.distributed as dist
    import paper_2402_00518_b200 as ee
    ee.load()
    store = dist.TCPStore("127.0.0.1", port, world, rank == 0, timeout=timedelta(seconds=60))
    cfg = _cfg("mlp", 90)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    N = targets.numel()
    nl = N // world
    c, prm, grd, ws, hid = _rank_setup(ee, cfg, mode, world, rank, params, hidden, "uniform")
    comm = ee.Comm(c, mode, world, rank, nl, exchange=ee.store_exchange(store, rank, world, mode))
    tg = targets[rank * nl:(rank + 1) * nl].cuda().contiguous()
    loss = torch.zeros(cfg.exits, device="cuda")
    ee.ee_tune_step(c, hid, tg, [1.0, 0.5], prm, grd, loss, ws, comm=comm)
    torch.cuda.synchronize()
    st = ee.ee_get_status(ws)
    ee.store_exchange(store, rank, world, mode + "/done")(0)   # peers done reading my arena
    comm.close()
    torch.save({"loss": loss.cpu(), "grads": [{k: v.cpu() for k, v in g.items()} for g in grd],
                "status": st}, f"{path}.{rank}")


@pytest.mark.parametrize("mode", ["dp", "vp"])
def test_comm_two_processes_tcpstore_only(gpu_lib, tmp_path, mode):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "out")
    mp.start_processes(_store_worker, args=(2, port, path, mode), nprocs=2, join=True,
                       start_method="spawn")
    outs = [torch.load(f"{path}.{r}") for r in range(2)]
    cfg = _cfg("mlp", 90)
    hidden = S.hidden_states(cfg)
    targets = S.targets(cfg)
    params = S.head_params(cfg)
    out = [(o["loss"], o["grads"], o["status"]) for o in outs]
    _check_vs_oracle(cfg, mode, 2, out, hidden, targets, params, [1.0, 0.5])
