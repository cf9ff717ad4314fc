"""Vocab-parallel orchestration on CPUs: world size 2 (and 3), gloo backend.

The product's vocab_parallel_step (paper_2402_00518_b200.parallel) runs over
real torch.distributed collectives (all-gather, signed-int64 MAX all-reduce of
the (max, argmax) key, SUM all-reduce, reduce-scatter); each rank's compute is
a numpy stand-in for the five ee_vp_* phases built from the fp64 oracle's
pieces.  Gathered W_out shards, all-reduced body grads, losses and argmax must
equal the single-process oracle on the full batch."""

import os
import socket
import struct

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


def _key(m, idx):
    """Same ordering as the CUDA key: orderable float32(m) high, ~idx low, sign-flipped."""
    u = struct.unpack("<I", struct.pack("<f", float(m)))[0]
    u = (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)
    k = (u << 32) | (0xFFFFFFFF - idx)
    k ^= 1 << 63
    return k - (1 << 64) if k >= 1 << 63 else k


def _unkey(k):
    k = (k + (1 << 64)) % (1 << 64)
    k ^= 1 << 63
    u = k >> 32
    u = (u & 0x7FFFFFFF) if u & 0x80000000 else (~u & 0xFFFFFFFF)
    return struct.unpack("<f", struct.pack("<I", u))[0], 0xFFFFFFFF - (k & 0xFFFFFFFF)


class NumpyPhases:
    """fp64 stand-in for the ee_vp_* phases of one rank (shard [vb, ve))."""

    def __init__(self, O, arch, vb, ve, eps=1e-5, attn=None):
        self.O, self.arch, self.vb, self.ve, self.eps = O, arch, vb, ve, eps
        self.attn = attn

    def exit_forward(self, hidden, params, z_out, n_all):
        p = {k: v.numpy() for k, v in params.items()}
        self.act = self.O.exit_forward(self.arch, p, hidden.numpy(), self.eps, self.attn)
        z_out.copy_(torch.from_numpy(self.act["z"]))

    def vocab_stats(self, z_all, targets_all, params, key, sums):
        S = z_all.numpy() @ params["w_out"].numpy().T
        self.S = S
        m = S.max(axis=1)
        am = S.argmax(axis=1) + self.vb
        self.m_loc = m
        y = targets_all.numpy()
        own = (y >= self.vb) & (y < self.ve)
        sums[:, 0] = torch.from_numpy(np.exp(S - m[:, None]).sum(axis=1))
        tl = np.where(own, S[np.arange(len(y)), np.clip(y - self.vb, 0, S.shape[1] - 1)], 0.0)
        sums[:, 1] = torch.from_numpy(tl)
        key.copy_(torch.tensor([_key(a, int(b)) for a, b in zip(m, am)], dtype=torch.int64))

    def rescale(self, key, sums):
        mg = np.array([_unkey(int(k))[0] for k in key])
        self.m_glob = mg
        sums[:, 0] *= torch.from_numpy(np.exp(self.m_loc - mg))

    def vocab_backward(self, i, z_all, targets_all, key, sums, alpha, W, params, grads,
                       dz_partial, loss_slot, accumulate, aux=None):
        s = sums.numpy()
        lse = self.m_glob + np.log(s[:, 0])
        y = targets_all.numpy()
        valid = y != -1
        Wv = float(W.item())
        loss_slot[0] = float(np.sum(np.where(valid, lse - s[:, 1], 0.0)) / Wv)
        P = np.exp(self.S - lse[:, None])
        own = valid & (y >= self.vb) & (y < self.ve)
        P[np.nonzero(own)[0], y[own] - self.vb] -= 1.0
        dS = (alpha * valid / Wv)[:, None] * P
        grads["w_out"].copy_(torch.from_numpy(dS.T @ z_all.numpy()))
        if dz_partial is not None:
            dz_partial.copy_(torch.from_numpy(dS @ params["w_out"].numpy()))
        if aux is not None:
            aux["argmax"].copy_(torch.tensor([_unkey(int(k))[1] for k in key]))

    def exit_backward(self, hidden, params, dz_local, grads, accumulate, n_all):
        if self.arch == "embedding":
            return
        p = {k: v.numpy() for k, v in params.items()}
        for k, g in self.O.exit_body_backward(self.arch, p, self.act, dz_local.numpy()).items():
            grads[k].copy_(torch.from_numpy(g))


def _worker(rank, world, port, arch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ee_oracle as O
        from paper_2402_00518_b200.parallel import TorchComm, vocab_parallel_step
        rng = np.random.default_rng(1)
        h, V, F, N, E = 16, 40, 24, 12 * world, 2
        at = {"seq_len": 6, "n_heads": 2, "n_kv": 1, "theta": 10000.0} if arch == "layer" else None
        params = [{"w_out": rng.normal(0, .5, (V, h))} for _ in range(E)]
        for p in params:
            if arch != "embedding":
                p["g_f"] = 1 + .1 * rng.normal(size=h)
            if arch in ("mlp", "layer"):
                p.update(g_a=1 + .1 * rng.normal(size=h), w_gate=rng.normal(0, .5, (F, h)),
                         w_up=rng.normal(0, .5, (F, h)), w_down=rng.normal(0, .5, (h, F)))
            if arch == "layer":
                p.update(g_att=1 + .1 * rng.normal(size=h), w_q=rng.normal(0, .5, (h, h)),
                         w_k=rng.normal(0, .5, (h // 2, h)), w_v=rng.normal(0, .5, (h // 2, h)),
                         w_o=rng.normal(0, .5, (h, h)))
        xs = [rng.normal(size=(N, h)) for _ in range(E)]
        y = rng.integers(0, V, N)
        y[[1, 7]] = -1
        alphas = [1.0, 0.7]
        w = 16                                            # shard width (multiple of 8)
        vb, ve = min(V, rank * w), (V if rank == world - 1 else min(V, (rank + 1) * w))
        nl = N // world
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        prm = [{k: T(v[vb:ve] if k == "w_out" else v) for k, v in p.items()} for p in params]
        grd = [{k: torch.zeros_like(v) for k, v in p.items()} for p in prm]
        hid = [T(x[rank * nl:(rank + 1) * nl]) for x in xs]
        bufs = {"z_all": torch.zeros(N, h, dtype=torch.float64),
                "key": torch.zeros(N, dtype=torch.int64),
                "sums": torch.zeros(N, 2, dtype=torch.float64),
                "dz_partial": torch.zeros(N, h, dtype=torch.float64),
                "dz_local": torch.zeros(nl, h, dtype=torch.float64)}
        W = torch.tensor([int(np.sum(y != -1))])
        loss = torch.zeros(E, dtype=torch.float64)
        aux = [{"argmax": torch.zeros(N, dtype=torch.int64)} for _ in range(E)]
        vocab_parallel_step(NumpyPhases(O, arch, vb, ve, attn=at), TorchComm(), arch, hid,
                            torch.from_numpy(y), prm, grd, loss, alphas, W, bufs, aux=aux)
        gathered = [None] * world
        dist.all_gather_object(gathered, ([g["w_out"].numpy() for g in grd],))
        if rank == 0:
            full_l, full_g, full_st = O.tune_step(arch, params, xs, y, alphas, 1e-5, attn=at)
            ok = np.allclose(loss.numpy(), full_l, rtol=1e-10)
            for i in range(E):
                dw = np.concatenate([gathered[r][0][i] for r in range(world)])
                ok &= np.allclose(dw, full_g[i]["w_out"], rtol=1e-9, atol=1e-14)
                for k in full_g[i]:
                    if k != "w_out":
                        ok &= np.allclose(grd[i][k].numpy(), full_g[i][k], rtol=1e-9, atol=1e-14)
                ok &= np.array_equal(aux[i]["argmax"].numpy(), full_st[i]["argmax"])
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("arch,world", [("mlp", 2), ("norm", 3), ("embedding", 2), ("layer", 2)])
def test_vocab_parallel_gloo_matches_full_batch_oracle(arch, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, arch, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_key_encoding_orders_by_value_then_lowest_index():
    vals = [(-3.5, 7), (-3.5, 2), (0.0, 9), (1e-30, 4), (2.25, 100), (2.25, 3), (float("inf"), 0)]
    keys = [_key(m, i) for m, i in vals]
    order = sorted(range(len(vals)), key=lambda j: keys[j])
    expect = sorted(range(len(vals)), key=lambda j: (vals[j][0], -vals[j][1]))
    assert order == expect
    for (m, i), k in zip(vals, keys):
        assert _unkey(k) == (np.float32(m), i)


# ---------------------------------------------------------------------------
# fused variant (vocab_parallel_step_fused): the host orchestration of the
# peer-memory all-gather / reduce-scatter, with shared-memory CPU tensors as
# the peers' buffers and gloo barriers as ee_peer_barrier
# ---------------------------------------------------------------------------

class SharedPeer:
    """CPU stand-in of parallel.PeerBuffers: z_all and the dz slots of every
    rank live in shared memory, so a rank's "NVLink stores" are plain writes."""

    def __init__(self, rank, world, z_tabs, slot_tabs):
        self.rank, self.world = rank, world
        self.z_tabs, self.slot_tabs = z_tabs, slot_tabs
        self.z_all = z_tabs[rank]
        self.slots = slot_tabs[rank]
        self.n_all = self.z_all.shape[0]
        self.n_local = self.n_all // world
        self.epoch = 0


class NumpyFusedPhases(NumpyPhases):
    def exit_forward_ag(self, hidden, params, peer, n_all):
        p = {k: v.numpy() for k, v in params.items()}
        self.act = self.O.exit_forward(self.arch, p, hidden.numpy(), self.eps, self.attn)
        z = torch.from_numpy(self.act["z"])
        r0 = peer.rank * peer.n_local
        for t in peer.z_tabs:                         # the all-gather: stores into every rank
            t[r0:r0 + peer.n_local].copy_(z)

    def vocab_backward_rs(self, i, z_all, targets_all, key, sums, alpha, W, params, grads, peer,
                          loss_slot, accumulate, aux=None):
        dz = torch.zeros(peer.n_all, z_all.shape[1], dtype=torch.float64)
        self.vocab_backward(i, z_all, targets_all, key, sums, alpha, W, params, grads,
                            None if self.arch == "embedding" else dz, loss_slot, accumulate, aux)
        if self.arch != "embedding":                  # the reduce-scatter: rows to their owners
            nl = peer.n_local
            for q in range(peer.world):
                peer.slot_tabs[q][peer.rank].copy_(dz[q * nl:(q + 1) * nl])

    def exit_backward_slots(self, hidden, params, peer, grads, accumulate, n_all):
        dz = peer.slots[0].clone()
        for q in range(1, peer.world):                # owner-side sum in rank order
            dz += peer.slots[q]
        self.exit_backward(hidden, params, dz, grads, accumulate, n_all)

    def barrier(self, peer):
        peer.epoch += 1
        dist.barrier()


def _fused_worker(rank, world, port, arch, z_tabs, slot_tabs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ee_oracle as O
        from paper_2402_00518_b200.parallel import TorchComm, vocab_parallel_step_fused
        rng = np.random.default_rng(2)
        h, V, F, N, E = 16, 40, 24, z_tabs[0].shape[0], 2
        params = [{"w_out": rng.normal(0, .5, (V, h))} for _ in range(E)]
        for p in params:
            if arch != "embedding":
                p["g_f"] = 1 + .1 * rng.normal(size=h)
            if arch == "mlp":
                p.update(g_a=1 + .1 * rng.normal(size=h), w_gate=rng.normal(0, .5, (F, h)),
                         w_up=rng.normal(0, .5, (F, h)), w_down=rng.normal(0, .5, (h, F)))
        xs = [rng.normal(size=(N, h)) for _ in range(E)]
        y = rng.integers(0, V, N)
        y[[0, 5]] = -1
        alphas = [1.0, 0.4]
        w = 16
        vb, ve = min(V, rank * w), (V if rank == world - 1 else min(V, (rank + 1) * w))
        nl = N // world
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        prm = [{k: T(v[vb:ve] if k == "w_out" else v) for k, v in p.items()} for p in params]
        grd = [{k: torch.zeros_like(v) for k, v in p.items()} for p in prm]
        hid = [T(x[rank * nl:(rank + 1) * nl]) for x in xs]
        bufs = {"key": torch.zeros(N, dtype=torch.int64),
                "sums": torch.zeros(N, 2, dtype=torch.float64)}
        W = torch.tensor([int(np.sum(y != -1))])
        loss = torch.zeros(E, dtype=torch.float64)
        peer = SharedPeer(rank, world, z_tabs, slot_tabs)
        ph = NumpyFusedPhases(O, arch, vb, ve)
        for _ in range(2):                            # twice: buffer reuse across steps
            vocab_parallel_step_fused(ph, TorchComm(), peer, arch, hid, torch.from_numpy(y), prm,
                                      grd, loss, alphas, W, bufs)
        gathered = [None] * world
        dist.all_gather_object(gathered, ([g["w_out"].numpy() for g in grd],))
        if rank == 0:
            full_l, full_g, _ = O.tune_step(arch, params, xs, y, alphas, 1e-5)
            ok = np.allclose(loss.numpy(), full_l, rtol=1e-10)
            ok &= peer.epoch == 2 * (1 + 2 * E)       # barriers per step: 1 + 2 per exit
            for i in range(E):
                dw = np.concatenate([gathered[r][0][i] for r in range(world)])
                ok &= np.allclose(dw, full_g[i]["w_out"], rtol=1e-9, atol=1e-14)
                for k in full_g[i]:
                    if k != "w_out":
                        ok &= np.allclose(grd[i][k].numpy(), full_g[i][k], rtol=1e-9, atol=1e-14)
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("arch,world", [("mlp", 2), ("norm", 3), ("embedding", 2)])
def test_fused_vocab_parallel_gloo_matches_full_batch_oracle(arch, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    N, h = 12 * world, 16
    z_tabs = [torch.zeros(N, h, dtype=torch.float64).share_memory_() for _ in range(world)]
    slot_tabs = [torch.zeros(world, N // world, h, dtype=torch.float64).share_memory_()
                 for _ in range(world)]
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, arch, z_tabs, slot_tabs, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_fused_orchestration_with_sharded_body_call_order():
    """vocab_parallel_step_fused(..., body=...) (ShardedVPHeads): per exit the
    body backward writes to the body's arenas (no local gradients, no body
    all-reduce), then one more peer barrier, then body.update(i); the step
    starts with one barrier.  Host logic only (recording stand-ins)."""
    from paper_2402_00518_b200.parallel import vocab_parallel_step_fused

    log = []

    class Rec:
        def __getattr__(self, name):
            def f(*a, **k):
                log.append((name, k.get("grad_arenas")))
            return f

        def barrier(self, peer):
            log.append(("barrier", None))

    class Comm:
        rank, world = 0, 1

        def all_reduce(self, t, op="sum", async_op=False):
            log.append(("all_reduce_" + op, None))

    class Body:
        def arena_set(self, i):
            return f"arena{i % 2}"

        def update(self, i):
            log.append(("update", i))

    class Peer:
        n_all, z_all = 8, None

    E = 3
    vocab_parallel_step_fused(Rec(), Comm(), Peer(), "mlp", [None] * E, None,
                              [{}] * E, [{"g_a": object()}] * E, torch.zeros(E), [1.0] * E,
                              None, {"key": None, "sums": None}, body=Body())
    names = [n for n, _ in log]
    assert names[0] == "barrier"
    per_exit = ["exit_forward_ag", "barrier", "vocab_stats", "all_reduce_max", "rescale",
                "all_reduce_sum", "vocab_backward_rs", "barrier", "exit_backward_slots",
                "barrier", "update"]
    assert names[1:] == per_exit * E, names
    arenas = [a for n, a in log if n == "exit_backward_slots"]
    assert arenas == ["arena0", "arena1", "arena0"]
    assert [x for n, x in log if n == "update"] == [0, 1, 2]
