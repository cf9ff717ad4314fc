"""Data-parallel host logic on CPUs: world size 2, gloo backend.

The product's DP orchestration (paper_2402_00518_b200.parallel) runs with the
fp64 oracle as each rank's compute; the all-reduced gradients and losses must
equal the single-process oracle on the full batch (P10), with the global
valid-token count used for normalisation (A16)."""

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


def _worker(rank, world, port, q, arch="mlp", weighting="uniform"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ee_oracle as O
        from paper_2402_00518_b200.parallel import data_parallel_step, shard_range
        rng = np.random.default_rng(0)
        h, V, F, N, E = 16, 40, 24, 37, 2
        T, align, at = 1, 1, None
        if arch == "layer":      # 7 sequences of 5 tokens, sharded as whole sequences
            T, N = 5, 35
            align = T
            at = {"seq_len": T, "n_heads": 2, "n_kv": 1, "theta": 10000.0}
        params = [{"w_out": rng.normal(0, .5, (V, h)), "g_f": 1 + .1 * rng.normal(size=h),
                   "g_a": 1 + .1 * rng.normal(size=h), "w_gate": rng.normal(0, .5, (F, h)),
                   "w_up": rng.normal(0, .5, (F, h)), "w_down": rng.normal(0, .5, (h, F))}
                  for _ in range(E)]
        if arch == "layer":
            for p in params:
                p.update(g_att=1 + .1 * rng.normal(size=h), w_q=rng.normal(0, .5, (h, h)),
                         w_k=rng.normal(0, .5, (h // 2, h)), w_v=rng.normal(0, .5, (h // 2, h)),
                         w_o=rng.normal(0, .5, (h, h)))
        xs = [rng.normal(size=(N, h)) for _ in range(E)]
        y = rng.integers(0, V, N)
        y[[1, 8, 30]] = -1
        alphas = [1.0, 0.6]
        s, e = shard_range(N, rank, world, align)
        grads = [{k: torch.zeros(v.shape, dtype=torch.float64) for k, v in p.items()} for p in params]
        loss = torch.zeros(E, dtype=torch.float64)

        def count_local():
            return torch.tensor([int(np.sum(y[s:e] != -1))], dtype=torch.int64)

        conf = weighting == "confidence"
        wsums = torch.zeros(E, dtype=torch.float64) if conf else None

        def run_exit(i, W):
            if not conf:
                r = O.exit_loss_and_grads(arch, params[i], xs[i][s:e], y[s:e], alphas[i], 1e-5,
                                          valid_count=int(W.item()), attn=at)
                loss[i] = r.loss
                for k, g in r.grads.items():
                    grads[i][k].copy_(torch.from_numpy(g))
                return
            # stand-in for EE_WEIGHT_CONFIDENCE_SUM: the locally normalised oracle
            # times the local sum of c_t (detached confidences of valid tokens)
            r = O.exit_loss_and_grads(arch, params[i], xs[i][s:e], y[s:e], alphas[i], 1e-5,
                                      weighting="confidence", attn=at)
            C = float(np.sum(r.stats["conf"][r.stats["valid"]]))
            wsums[i] = C
            loss[i] = r.loss * C
            for k, g in r.grads.items():
                grads[i][k].copy_(torch.from_numpy(g * C))

        def normalize(i):
            loss[i] /= wsums[i]
            for g in grads[i].values():
                g /= wsums[i]

        W = data_parallel_step(E, None if conf else count_local, run_exit,
                               lambda i: grads[i].values(), loss, weight_sums=wsums,
                               normalize=normalize)
        if rank == 0:
            if conf:
                full_l, full_g = [], []
                for i in range(E):
                    r = O.exit_loss_and_grads(arch, params[i], xs[i], y, alphas[i], 1e-5,
                                              weighting="confidence", attn=at)
                    full_l.append(r.loss)
                    full_g.append(r.grads)
                full_l = np.array(full_l)
                ok = True
            else:
                full_l, full_g, _ = O.tune_step(arch, params, xs, y, alphas, 1e-5, attn=at)
                ok = int(W.item()) == int(np.sum(y != -1))
            ok &= np.allclose(loss.numpy(), full_l, rtol=1e-12)
            for i in range(E):
                for k in params[i]:
                    ok &= np.allclose(grads[i][k].numpy(), full_g[i][k], rtol=1e-10, atol=1e-15)
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("arch,weighting", [("mlp", "uniform"), ("layer", "uniform"),
                                            ("mlp", "confidence")])
def test_data_parallel_world2_matches_full_batch_oracle(arch, weighting):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, arch, weighting)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_shard_range_covers_tokens():
    from paper_2402_00518_b200.parallel import shard_range
    for n in (0, 1, 7, 65536, 65539):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    for w in (1, 2, 3):                                 # whole sequences (Layer exits)
        spans = [shard_range(7 * 2048, r, w, 2048) for r in range(w)]
        assert spans[-1][1] == 7 * 2048 and all(a % 2048 == 0 and b % 2048 == 0 for a, b in spans)
    with pytest.raises(ValueError):
        shard_range(100, 0, 2, 64)
