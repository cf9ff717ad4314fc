"""Fused vocab-parallel collectives over peer memory (include/ee.h
ee_vp_exit_forward_ag / ee_vp_vocab_backward_rs / ee_vp_exit_backward_slots /
ee_peer_barrier; parallel.vocab_parallel_step_fused) on one GPU.

1. P ranks emulated by P host threads, each on its OWN CUDA stream, so the
   ranks' kernels run concurrently and the device barrier (ee_peer_barrier)
   really synchronises them; the peer pointer tables point at the other
   threads' buffers.  Results must equal the NCCL-style path
   (vocab_parallel_step with rank-ordered host collectives) BIT FOR BIT -- the
   fused reduce-scatter sums the slots in the same rank order -- and the fp64
   oracle within north_star tolerances.
2. Two processes on the same GPU, buffers mapped with CUDA IPC
   (ee_ipc_get_handle / ee_ipc_open, handles exchanged over gloo): the
   production connect_ipc path end to end against the oracle.
"""

import os
import threading

import numpy as np
import pytest
import torch

import eesynth as S
from harness import GRAD_RTOL, grad_rtol, LOSS_RTOL, attn_kwargs, oracle_exit, rel_fro

pytestmark = pytest.mark.gpu


class StreamThreadComm:
    """In-process collectives for ranks on their own streams (rank-ordered
    sums, like tests/test_gpu_vp.py's ThreadComm) that synchronise only the
    caller's stream, never the device: a rank blocked here must not wait for
    another rank's spinning barrier kernel."""

    def __init__(self, shared, rank, stream):
        self.s, self.rank, self.world, self.stream = shared, rank, shared["P"], stream

    def _exchange(self, t):
        self.stream.synchronize()
        with torch.cuda.stream(self.stream):
            c = t.detach().clone()
        self.stream.synchronize()
        self.s["slots"][self.rank] = c
        self.s["barrier"].wait()
        vals = list(self.s["slots"])
        self.s["barrier"].wait()
        return vals

    def all_gather_into(self, out, inp):
        vals = self._exchange(inp)
        with torch.cuda.stream(self.stream):
            out.copy_(torch.cat(vals))

    def all_reduce(self, t, op="sum", async_op=False):
        vals = self._exchange(t)
        with torch.cuda.stream(self.stream):
            if op == "max":
                res = torch.stack(vals).max(dim=0).values
            else:
                res = vals[0].clone()
                for v in vals[1:]:
                    res += v
            t.copy_(res)
        return None

    def reduce_scatter(self, out, inp):
        vals = self._exchange(inp)
        with torch.cuda.stream(self.stream):
            tot = vals[0].clone()
            for v in vals[1:]:
                tot += v
            n = out.shape[0]
            out.copy_(tot[self.rank * n:(self.rank + 1) * n])


def _rank_inputs(ee, cfg, P, r, params, hidden, targets, N, weighting="uniform"):
    from paper_2402_00518_b200.parallel import vocab_shard
    vb, ve = vocab_shard(cfg.vocab, P, r)
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, cfg.exits, cfg.arch, 1e-5, vb, ve,
                       token_weighting=weighting, **attn_kwargs(cfg))
    ws = torch.zeros(ee.ee_workspace_size(c, N), dtype=torch.uint8, device="cuda")
    prm, grd = [], []
    for p in params:
        d = {}
        for k, v in p.items():
            v = v[vb:ve] if k == "w_out" else v
            d[k] = v.cuda().float().contiguous() if k.startswith("g_") else \
                v.cuda().to(torch.bfloat16).contiguous()
        prm.append(d)
        grd.append({k: torch.full(d[k].shape, float("nan"), device="cuda") for k in d})
    nl = N // P
    hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
    return c, ws, prm, grd, hid


def run_threads(ee, cfg, P, hidden, targets, params, weights, fused, steps=1):
    from paper_2402_00518_b200.parallel import (GpuPhases, PeerBuffers, vocab_parallel_step,
                                                vocab_parallel_step_fused)
    N, h, E = targets.numel(), cfg.hidden, cfg.exits
    nl = N // P
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": [None] * P}
    tg = targets.cuda()
    peers = [PeerBuffers(r, P, N, h) for r in range(P)] if fused else None
    if fused:
        for b in peers:
            b.connect_local(peers)
    torch.cuda.synchronize()
    out, errors = [None] * P, []

    def rank_fn(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                c, ws, prm, grd, hid = _rank_inputs(ee, cfg, P, r, params, hidden, targets, N)
                bufs = {"z_all": torch.zeros(N, h, dtype=torch.bfloat16, device="cuda"),
                        "key": torch.zeros(N, dtype=torch.int64, device="cuda"),
                        "sums": torch.zeros(N, 2, device="cuda"),
                        "dz_partial": torch.zeros(N, h, device="cuda"),
                        "dz_local": torch.zeros(nl, h, device="cuda")}
                W = torch.tensor([int((targets != -1).sum())], dtype=torch.int64, device="cuda")
                loss = torch.zeros(E, device="cuda")
                comm = StreamThreadComm(shared, r, st)
                ph = GpuPhases(ee, c, ws, stream=st)
                for _ in range(steps):
                    if fused:
                        vocab_parallel_step_fused(ph, comm, peers[r], cfg.arch, hid, tg, prm, grd,
                                                  loss, weights, W, bufs)
                    else:
                        vocab_parallel_step(ph, comm, cfg.arch, hid, tg, prm, grd, loss, weights,
                                            W, bufs)
                st.synchronize()
                out[r] = (loss.cpu(), [{k: v.cpu() for k, v in g.items()} for g in grd],
                          ee.ee_get_status(ws, stream=st))
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


def _cfg(arch, seed):
    if arch == "layer":     # 2 sequences of 128: one per rank
        return S.get_cfg("tiny_layer", seed=seed)
    return S.Cfg(name="small", hidden=128, vocab=1000, ffn=256 if arch == "mlp" else 0,
                 arch=arch, tokens=256, layers=2, after=[1, 2], init="random", seed=seed)


@pytest.mark.parametrize("arch,P", [("mlp", 2), ("mlp", 4), ("norm", 4), ("embedding", 2),
                                    ("layer", 2), ("mlp", 8)])
def test_fused_vp_bitwise_equals_nccl_path_and_matches_oracle(gpu_lib, arch, P):
    cfg = _cfg(arch, 31)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    weights = [1.0, 0.5]
    ref = run_threads(gpu_lib, cfg, P, hidden, targets, params, weights, fused=False)
    fus = run_threads(gpu_lib, cfg, P, hidden, targets, params, weights, fused=True, steps=2)
    for r in range(P):
        assert fus[r][2] == (0, -1), fus[r][2]
        assert torch.equal(fus[r][0], ref[r][0])
        for i in range(cfg.exits):
            for k, g in ref[r][1][i].items():
                assert torch.equal(fus[r][1][i][k], g), (r, i, k)
    for i in range(cfg.exits):
        res = oracle_exit(arch, params[i], hidden[i], targets, weights[i],
                          attn=S.attn_geometry(cfg))
        assert abs(fus[0][0][i].item() - res.loss) / res.loss <= LOSS_RTOL
        dw = torch.cat([fus[r][1][i]["w_out"] for r in range(P)]).double().numpy()
        assert rel_fro(dw, res.grads["w_out"]) <= GRAD_RTOL
        for k in res.grads:
            if k != "w_out":
                assert rel_fro(fus[0][1][i][k].double().numpy(), res.grads[k]) <= grad_rtol(cfg.arch, k), k


def test_peer_barrier_reports_missing_peer(gpu_lib):
    """A peer that never arrives: the barrier gives up after its timeout and
    sets EE_ERR_PEER (code 12, exit_index = the missing rank) -- no hang."""
    ee = gpu_lib
    sig = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(2)]
    ws = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    ee.ee_peer_barrier(ee.peer_set(0, sig), 1, ws)
    torch.cuda.synchronize()
    assert ee.ee_get_status(ws) == (12, 1)
    assert sig[1][0].item() == 1                 # rank 0's arrival was published to rank 1


# ---------------------------------------------------------------------------
# two processes, one GPU, CUDA IPC
# ---------------------------------------------------------------------------

class GlooComm:
    """CE-statistics and gradient collectives over gloo (host staging)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist, self.rank, self.world = dist, dist.get_rank(), dist.get_world_size()

    def all_reduce(self, t, op="sum", async_op=False):
        c = t.cpu()
        self.dist.all_reduce(c, op=self.dist.ReduceOp.MAX if op == "max" else
                             self.dist.ReduceOp.SUM)
        t.copy_(c)
        return None


def _ipc_worker(rank, world, port, path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2402_00518_b200 as ee
    from paper_2402_00518_b200.parallel import GpuPhases, PeerBuffers, vocab_parallel_step_fused
    ee.load()
    cfg = _cfg("mlp", 41)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    N = targets.numel()
    c, ws, prm, grd, hid = _rank_inputs(ee, cfg, world, rank, params, hidden, targets, N)
    peer = PeerBuffers(rank, world, N, cfg.hidden)
    torch.cuda.synchronize()
    peer.connect_ipc()
    bufs = {"key": torch.zeros(N, dtype=torch.int64, device="cuda"),
            "sums": torch.zeros(N, 2, device="cuda")}
    W = torch.tensor([int((targets != -1).sum())], dtype=torch.int64, device="cuda")
    loss = torch.zeros(cfg.exits, device="cuda")
    vocab_parallel_step_fused(GpuPhases(ee, c, ws), GlooComm(), peer, cfg.arch, hid,
                              targets.cuda(), prm, grd, loss, [1.0, 0.5], W, bufs)
    torch.cuda.synchronize()
    st = ee.ee_get_status(ws)
    dist.barrier()
    peer.close()
    torch.save({"loss": loss.cpu(), "grads": [{k: v.cpu() for k, v in g.items()} for g in grd],
                "status": st}, f"{path}.{rank}")
    dist.destroy_process_group()


def test_fused_vp_two_processes_cuda_ipc(gpu_lib, tmp_path):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "out")
    mp.start_processes(_ipc_worker, args=(2, port, path), nprocs=2, join=True,
                       start_method="spawn")
    outs = [torch.load(f"{path}.{r}") for r in range(2)]
    cfg = _cfg("mlp", 41)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    for o in outs:
        assert o["status"] == (0, -1)
    for i, a in enumerate([1.0, 0.5]):
        res = oracle_exit("mlp", params[i], hidden[i], targets, a)
        for o in outs:
            assert abs(o["loss"][i].item() - res.loss) / res.loss <= LOSS_RTOL
        dw = torch.cat([o["grads"][i]["w_out"] for o in outs]).double().numpy()
        assert rel_fro(dw, res.grads["w_out"]) <= GRAD_RTOL
        for k in ("g_a", "w_gate", "w_up", "w_down", "g_f"):
            for o in outs:
                assert rel_fro(o["grads"][i][k].double().numpy(), res.grads[k]) <= grad_rtol(cfg.arch, k), k


# ---------------------------------------------------------------------------
# sharded exit-body update under VP (ShardedVPHeads, body=...)
# ---------------------------------------------------------------------------

def _run_vp_adam(ee, cfg, P, hidden, targets, params, sharded, steps=2):
    from paper_2402_00518_b200.parallel import (GpuPhases, PeerBuffers, ShardedVPHeads,
                                                vocab_parallel_step_fused, vocab_shard)
    N, h, E = targets.numel(), cfg.hidden, cfg.exits
    nl = N // P
    kw = attn_kwargs(cfg)
    spec = ee.HeadSpec(h, cfg.vocab, cfg.ffn, E, cfg.arch, **kw)
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": [None] * P}
    peers = [PeerBuffers(r, P, N, h) for r in range(P)]
    for b in peers:
        b.connect_local(peers)
    zs = [ShardedVPHeads(spec, N, r, P) for r in range(P)] if sharded else None
    if sharded:
        for z in zs:
            z.connect_local(zs)
    torch.cuda.synchronize()
    tg = targets.cuda()
    out, errors = [None] * P, []

    def src(r):
        vb, ve = vocab_shard(cfg.vocab, P, r)
        return [{k: (v[vb:ve] if k == "w_out" else v).cuda().float().contiguous()
                 for k, v in p.items()} for p in params]

    def rank_fn(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = StreamThreadComm(shared, r, st)
                hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
                bufs = {"key": torch.zeros(N, dtype=torch.int64, device="cuda"),
                        "sums": torch.zeros(N, 2, device="cuda")}
                W = torch.tensor([int((targets != -1).sum())], dtype=torch.int64, device="cuda")
                vb, ve = vocab_shard(cfg.vocab, P, r)
                if sharded:
                    hd = zs[r]
                    hd.init("copy", copy_src=src(r), src_dtype=torch.float32)
                    ph = GpuPhases(ee, hd.exit_cfg, hd.workspace, stream=st)
                    for it in range(steps):
                        hd.set_lr(1e-3 * (it + 1))
                        vocab_parallel_step_fused(ph, comm, peers[r], cfg.arch, hid, tg,
                                                  hd.operand, hd.grads, hd.loss, [1.0, 0.5], W,
                                                  bufs, body=hd)
                    layout = hd.layout
                else:
                    hd = ee.ExitHeads(ee.HeadSpec(h, cfg.vocab, cfg.ffn, E, cfg.arch,
                                                  vocab_begin=vb, vocab_end=ve, **kw), N)
                    hd.init("copy", copy_src=src(r), src_dtype=torch.float32)
                    ph = GpuPhases(ee, hd.exit_cfg, hd.workspace, stream=st)
                    for it in range(steps):
                        vocab_parallel_step_fused(ph, comm, peers[r], cfg.arch, hid, tg,
                                                  hd.operand, hd.grads, hd.loss, [1.0, 0.5], W,
                                                  bufs)
                        hd.adam(1e-3 * (it + 1))
                    layout = None
                st.synchronize()
                out[r] = ([{k: v.cpu() for k, v in d.items()} for d in hd.operand],
                          [{k: v.cpu() for k, v in d.items()} for d in hd.master], layout,
                          hd.loss.cpu(), ee.ee_get_status(hd.workspace, stream=st))
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


@pytest.mark.parametrize("arch,P", [("mlp", 2), ("mlp", 4), ("embedding", 2), ("norm", 4),
                                    ("layer", 2)])
def test_vp_sharded_body_update_bitwise(gpu_lib, arch, P):
    """VP with the exit body's gradient rows scattered to their owners and a
    sharded Adam (ZeRO-1 for the replicated body) equals, bit for bit, the
    fused VP step with the rank-ordered body all-reduce and a full Adam on
    every rank: all operands on every rank, the W_out shard's master, the
    body master rows each rank owns."""
    cfg = _cfg(arch, 37)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    _warm_vp = _run_vp_adam(gpu_lib, cfg, 1, hidden, targets, params, sharded=True, steps=1)
    ref = _run_vp_adam(gpu_lib, cfg, P, hidden, targets, params, sharded=False)
    got = _run_vp_adam(gpu_lib, cfg, P, hidden, targets, params, sharded=True)
    for r in range(P):
        assert got[r][4] == (0, -1), got[r][4]
        assert torch.equal(got[r][3], ref[r][3])
        for i in range(cfg.exits):
            for k, t in ref[r][0][i].items():
                assert torch.equal(got[r][0][i][k], t), (r, i, k, "operand")
            for k, full in ref[r][1][i].items():
                if k == "w_out":
                    assert torch.equal(got[r][1][i][k], full), (r, i, k)
                    continue
                b, rows = got[r][2][k][0], got[r][2][k][1]
                want = full.reshape(-1, full.shape[-1])[b:b + rows]
                assert torch.equal(got[r][1][i][k], want), (r, i, k)
