"""Vocab-parallel W_out on one GPU: P ranks emulated by P host threads, each
driving the CUDA ee_vp_* phases through the product orchestration
(paper_2402_00518_b200.parallel.vocab_parallel_step) with an in-process
collective (ThreadComm: barrier + exchange of device tensors, rank-ordered
sums).  The gathered W_out shards, the all-reduced exit-body gradients and the
loss must match the fp64 oracle on the full batch (north_star tolerances).
The NCCL transport itself is exercised on CPUs by tests/test_vp_gloo.py."""

import threading

import numpy as np
import pytest
import torch

import eesynth as S
from harness import GRAD_RTOL, grad_rtol, LOSS_RTOL, attn_kwargs, check_argmax, oracle_exit, rel_fro

pytestmark = pytest.mark.gpu


class ThreadComm:
    def __init__(self, shared, rank):
        self.s, self.rank, self.world = shared, rank, shared["P"]

    def _exchange(self, t):
        torch.cuda.synchronize()
        self.s["slots"][self.rank] = t.detach().clone()
        self.s["barrier"].wait()
        vals = list(self.s["slots"])
        self.s["barrier"].wait()
        return vals

    def all_gather_into(self, out, inp):
        vals = self._exchange(inp)
        out.copy_(torch.cat(vals))

    def all_reduce(self, t, op="sum", async_op=False):
        vals = self._exchange(t)
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
        tot = vals[0].clone()
        for v in vals[1:]:
            tot += v
        n = out.shape[0]
        out.copy_(tot[self.rank * n:(self.rank + 1) * n])


def _shards(V, P):
    """Contiguous vocab shards whose widths are multiples of 8 (ragged last)."""
    w = ((V // P + 7) // 8) * 8
    edges = [min(V, r * w) for r in range(P)] + [V]
    return [(edges[r], edges[r + 1]) for r in range(P)]


def run_vp(ee, cfg, P, hidden, targets, params, weights, weighting="uniform"):
    from paper_2402_00518_b200.parallel import GpuPhases, vocab_parallel_step
    N, h, E = targets.numel(), cfg.hidden, cfg.exits
    nl = N // P
    shards = _shards(cfg.vocab, P)
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": [None] * P}
    tg = targets.cuda()
    out = [None] * P
    errors = []

    def rank_fn(r):
        try:
            vb, ve = shards[r]
            c = ee.make_config(h, cfg.vocab, cfg.ffn, E, cfg.arch, 1e-5, vb, ve,
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
            hid = [x[r * nl:(r + 1) * nl].cuda().contiguous() for x in hidden]
            bufs = {"z_all": torch.zeros(N, h, dtype=torch.bfloat16, device="cuda"),
                    "key": torch.zeros(N, dtype=torch.int64, device="cuda"),
                    "sums": torch.zeros(N, 2, device="cuda"),
                    "dz_partial": torch.zeros(N, h, device="cuda"),
                    "dz_local": torch.zeros(nl, h, device="cuda")}
            W = torch.tensor([int((targets != -1).sum())], dtype=torch.int64, device="cuda")
            loss = torch.zeros(E, device="cuda")
            aux = [{"lse": torch.zeros(N, device="cuda"),
                    "argmax": torch.zeros(N, dtype=torch.int32, device="cuda")} for _ in range(E)]
            vocab_parallel_step(GpuPhases(ee, c, ws), ThreadComm(shared, r), cfg.arch, hid, tg,
                                prm, grd, loss, weights, W, bufs, aux=aux)
            torch.cuda.synchronize()
            out[r] = (loss.cpu(), [{k: v.cpu() for k, v in g.items()} for g in grd],
                      [{k: v.cpu() for k, v in a.items()} for a in aux], ee.ee_get_status(ws))
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
    return out, shards


@pytest.mark.parametrize("arch,P", [("mlp", 2), ("mlp", 4), ("norm", 4), ("embedding", 2),
                                    ("layer", 2)])
def test_vocab_parallel_matches_oracle(gpu_lib, arch, P):
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256 if arch == "mlp" else 0,
                arch=arch, tokens=256, layers=2, after=[1, 2], init="random", seed=21)
    if arch == "layer":     # 2 sequences of 128: one per rank
        cfg = S.get_cfg("tiny_layer", seed=21)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    weights = [1.0, 0.5]
    out, shards = run_vp(gpu_lib, cfg, P, hidden, targets, params, weights)
    for r in range(P):
        assert out[r][3] == (0, -1)
    for i in range(cfg.exits):
        res = oracle_exit(arch, params[i], hidden[i], targets, weights[i],
                          attn=S.attn_geometry(cfg))
        for r in range(P):                                     # loss identical on every rank
            L = out[r][0][i].item()
            assert abs(L - res.loss) / res.loss <= LOSS_RTOL
            assert out[r][0][i].item() == out[0][0][i].item()
        dw = torch.cat([out[r][1][i]["w_out"] for r in range(P)]).double().numpy()
        assert rel_fro(dw, res.grads["w_out"]) <= GRAD_RTOL
        for k in res.grads:
            if k == "w_out":
                continue
            for r in range(P):                                 # all-reduced body grads
                assert rel_fro(out[r][1][i][k].double().numpy(), res.grads[k]) <= grad_rtol(cfg.arch, k), k
        lse = out[0][2][i]["lse"].double().numpy()
        assert np.max(np.abs(lse - res.stats["lse"])) <= 5e-2
        check_argmax(out[0][2][i]["argmax"].numpy(), res.act["S"])


def test_vocab_parallel_p1_equals_single_gpu_step(gpu_lib):
    """P = 1 through the phases reproduces ee_tune_step (same kernels, same
    order): bitwise-equal loss and gradients."""
    from harness import gpu_step
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=200,
                layers=2, after=[1], init="random", seed=22)
    hidden = S.hidden_states(cfg, 200)
    targets = S.targets(cfg, 200)
    params = S.head_params(cfg)
    out, _ = run_vp(gpu_lib, cfg, 1, hidden, targets, params, [1.0])
    loss, grads, aux, st = gpu_step(gpu_lib, cfg, hidden, targets, params, [1.0])
    assert out[0][0][0].item() == loss[0].item()
    for k, g in grads[0].items():
        assert torch.equal(out[0][1][0][k], g.cpu()), k


def test_vocab_parallel_confidence_weighting(gpu_lib):
    """Dynamic token weights under VP: every rank sees all tokens after the
    stats all-reduce, so sum_t c_t is formed locally (no extra collective)."""
    cfg = S.Cfg(name="small", hidden=128, vocab=1000, ffn=256, arch="mlp", tokens=256, layers=2,
                after=[1], init="random", seed=23)
    hidden = S.hidden_states(cfg, 256)
    targets = S.targets(cfg, 256)
    params = S.head_params(cfg)
    out, shards = run_vp(gpu_lib, cfg, 4, hidden, targets, params, [1.0], weighting="confidence")
    res = oracle_exit("mlp", params[0], hidden[0], targets, 1.0, weighting="confidence")
    assert abs(out[0][0][0].item() - res.loss) / res.loss <= LOSS_RTOL
    dw = torch.cat([out[r][1][0]["w_out"] for r in range(4)]).double().numpy()
    assert rel_fro(dw, res.grads["w_out"]) <= GRAD_RTOL
    for k in ("g_a", "w_gate", "w_up", "w_down", "g_f"):
        assert rel_fro(out[0][1][0][k].double().numpy(), res.grads[k]) <= grad_rtol(cfg.arch, k), k
