"""Forward-communication-only pipeline schedule (NEXT #3) on CPUs:
2 stages over gloo, fp64 oracle compute.  Stage s runs its backbone layers
forward per microbatch, sends the activation forward and tunes its own exits
immediately; the per-stage exit gradients (accumulated over microbatches with
the global valid count) equal the single-process oracle on the full batch."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(7)
    h, nh, nkv, F, V, T = 16, 2, 1, 24, 40, 5
    n_layers, micro, seqs_per_micro = 4, 3, 2
    layers = []
    for _ in range(n_layers):
        layers.append({"g_att": 1 + .1 * rng.normal(size=h), "w_q": rng.normal(0, .3, (h, h)),
                       "w_k": rng.normal(0, .3, (h // 2, h)), "w_v": rng.normal(0, .3, (h // 2, h)),
                       "w_o": rng.normal(0, .3, (h, h)), "g_mlp": 1 + .1 * rng.normal(size=h),
                       "w_gate": rng.normal(0, .3, (F, h)), "w_up": rng.normal(0, .3, (F, h)),
                       "w_down": rng.normal(0, .3, (h, F))})
    exits_after = [1, 2, 3, 4]                       # one MLP exit after every layer
    heads = [{"w_out": rng.normal(0, .5, (V, h)), "g_f": 1 + .1 * rng.normal(size=h),
              "g_a": 1 + .1 * rng.normal(size=h), "w_gate": rng.normal(0, .5, (F, h)),
              "w_up": rng.normal(0, .5, (F, h)), "w_down": rng.normal(0, .5, (h, F))}
             for _ in exits_after]
    N = micro * seqs_per_micro * T
    x0 = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    y[[2, 9, 17]] = -1
    return dict(h=h, nh=nh, nkv=nkv, T=T, layers=layers, exits_after=exits_after, heads=heads,
                x0=x0, y=y, micro=micro, mb=seqs_per_micro * T)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ee_oracle as O
        from paper_2402_00518_b200.parallel import TorchP2P, pipeline_forward_only_step
        P = _problem()
        L_per = len(P["layers"]) // world
        my_layers = range(rank * L_per + 1, (rank + 1) * L_per + 1)          # 1-based
        my_exits = [i for i, k in enumerate(P["exits_after"]) if k in my_layers]
        W = int(np.sum(P["y"] != -1))                                         # global valid count
        grads = {i: {k: np.zeros_like(v) for k, v in P["heads"][i].items()} for i in my_exits}
        losses = {i: 0.0 for i in my_exits}
        cache = {}

        def fwd(m, x_in):
            x = P["x0"][m * P["mb"]:(m + 1) * P["mb"]] if x_in is None else x_in.numpy()
            for l in my_layers:
                x = O.llama_layer_forward(P["layers"][l - 1], x, P["T"], P["nh"], P["nkv"], 1e-5)
                for i in my_exits:
                    if P["exits_after"][i] == l:
                        cache[(m, i)] = x.copy()
            return torch.from_numpy(x)

        def exits(m):
            ym = P["y"][m * P["mb"]:(m + 1) * P["mb"]]
            for i in my_exits:
                r = O.exit_loss_and_grads("mlp", P["heads"][i], cache.pop((m, i)), ym, 1.0, 1e-5,
                                          valid_count=W)
                losses[i] += r.loss
                for k, g in r.grads.items():
                    grads[i][k] += g

        p2p = TorchP2P(rank, (P["mb"], P["h"]), torch.float64, "cpu")
        pipeline_forward_only_step(rank, world, P["micro"], fwd, exits, p2p.send, p2p.recv)
        assert not cache                                  # no activations kept
        res = [None] * world
        dist.all_gather_object(res, (losses, grads))
        if rank == 0:
            hid = O.backbone_forward(P["layers"], P["x0"], P["T"], P["nh"], P["nkv"],
                                     P["exits_after"], 1e-5)
            full_l, full_g, _ = O.tune_step("mlp", P["heads"], hid, P["y"], [1.0] * 4, 1e-5)
            ok = True
            for r_ in range(world):
                L_r, G_r = res[r_]
                for i in L_r:
                    ok &= abs(L_r[i] - full_l[i]) <= 1e-12 * abs(full_l[i])
                    for k in G_r[i]:
                        ok &= np.allclose(G_r[i][k], full_g[i][k], rtol=1e-10, atol=1e-14)
            ok &= sorted(i for r_ in range(world) for i in res[r_][0]) == [0, 1, 2, 3]
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_forward_only_pipeline_two_stages_matches_full_batch_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
