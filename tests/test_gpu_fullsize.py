"""Full-size parity in the launch configuration bench.py times (BASELINE.json
configs at their full token counts, one exit = the same GEMM launches the
bench repeats per exit).  The oracle cannot run the full batch (~1e14 fp64
FLOPs), so these check (a) sampled rows the oracle computes one by one (lse,
loss_t, confidence, argmax), and (b) properties that hold at any size:
loss = mean of the per-token losses, softmax-CE gradient rows sum to zero
(P4), bitwise rerun determinism, read-only inputs, and -- for the Embedding
config, where z = x -- the uniform-logit closed form of dW_out (P3) on every
element."""

import math

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from harness import check_argmax
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


def _one_exit(name):
    cfg = S.get_cfg(name)
    cfg.after = cfg.after[:1]
    cfg.exits = 1
    return cfg


def _run(ee, cfg, hidden, targets, params, aux=True):
    n = targets.numel()
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, cfg.arch)
    ops = [{k: (v.float().contiguous() if k.startswith("g_") else v.to(torch.bfloat16).contiguous())
            for k, v in params[0].items()}]
    grads = [{k: torch.empty(v.shape, device="cuda") for k, v in params[0].items()}]
    ax = [{"lse": torch.zeros(n, device="cuda"), "loss_tok": torch.zeros(n, device="cuda"),
           "argmax": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "conf": torch.zeros(n, device="cuda")}]
    ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, device="cuda")
    ee.ee_tune_step(c, hidden, targets, [1.0], ops, grads, loss, ws, aux=ax)
    torch.cuda.synchronize()
    return loss, grads, ax, ee.ee_get_status(ws), ops


@pytest.mark.parametrize("name", ["13b", "70b"])
def test_full_size_sampled_rows_and_invariants(gpu_lib, name):
    ee = gpu_lib
    cfg = _one_exit(name)
    n = cfg.tokens
    hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
    targets = S.targets(cfg, n, device="cuda")
    params = S.head_params(cfg, device="cuda")
    h0 = hidden[0].clone()
    loss, grads, aux, st, ops = _run(ee, cfg, hidden, targets, params)
    assert st == (0, -1)
    assert torch.equal(hidden[0], h0)                                   # frozen input
    # (a) sampled rows vs the oracle, row by row
    tg = targets.cpu().numpy()
    rows = np.unique(np.concatenate([[0, 1, n // 2, n - 1], np.nonzero(tg == -1)[0][:2],
                                     np.random.default_rng(0).integers(0, n, 10)]))
    p64 = {k: to_f64(v) for k, v in ops[0].items()}
    act = O.exit_forward(cfg.arch, p64, to_f64(hidden[0][torch.as_tensor(rows, device="cuda")]),
                         1e-5)
    st_o = O.lm_loss_stats(act["S"], tg[rows])
    lse = aux[0]["lse"].cpu().numpy()[rows]
    assert np.max(np.abs(lse - st_o["lse"])) <= 5e-2
    assert np.max(np.abs(aux[0]["conf"].cpu().numpy()[rows] - st_o["conf"])) <= 2e-2
    lt = aux[0]["loss_tok"].cpu().numpy()[rows]
    assert np.max(np.abs(lt - st_o["loss"])) <= 5e-2
    assert np.all(lt[tg[rows] == -1] == 0.0)
    check_argmax(aux[0]["argmax"].cpu().numpy()[rows], act["S"])
    # (b) loss = mean of per-token losses over valid tokens
    valid = tg != -1
    lt_all = aux[0]["loss_tok"].double().cpu().numpy()
    assert abs(loss.item() - lt_all[valid].mean()) <= 1e-5 * abs(loss.item())
    # P4: sum_v dW_out[v, :] = 0 (dS rows sum to zero), against the no-cancellation scale
    dw = grads[0]["w_out"].double()
    colsum = dw.sum(dim=0).norm().item()
    scale = dw.abs().sum(dim=0).norm().item()
    assert colsum <= 1e-2 * scale, (colsum, scale)
    for k, g in grads[0].items():
        assert torch.isfinite(g).all(), k
    # bitwise rerun determinism (no float atomics anywhere)
    loss2, grads2, _, _, _ = _run(ee, cfg, hidden, targets, params)
    assert torch.equal(loss, loss2)
    for k in grads[0]:
        assert torch.equal(grads[0][k], grads2[0][k]), k


def test_full_size_embedding_uniform_logits_closed_form(gpu_lib):
    """7B config (Embedding exit, z = x), W_out = 0: loss = ln V, conf = 1/V and
    dW_out[v] = (1/W) sum_t w_t (1/V - 1[y_t = v]) x_t on every element (P3)."""
    ee = gpu_lib
    cfg = _one_exit("7b")
    n, V = cfg.tokens, cfg.vocab
    hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
    targets = S.targets(cfg, n, device="cuda")
    params = S.head_params(cfg, device="cuda")
    params[0]["w_out"].zero_()
    loss, grads, aux, st, _ = _run(ee, cfg, hidden, targets, params)
    assert st == (0, -1)
    assert abs(loss.item() - math.log(V)) <= 1e-5 * math.log(V)
    assert torch.allclose(aux[0]["conf"], torch.full_like(aux[0]["conf"], 1.0 / V), rtol=1e-5)
    x = to_f64(hidden[0])
    y = targets.cpu().numpy()
    w = (y != -1).astype(np.float64)
    W = w.sum()
    expect = np.tile((w @ x) / (V * W), (V, 1))
    np.subtract.at(expect, y[w > 0], x[w > 0] / W)
    got = grads[0]["w_out"].double().cpu().numpy()
    rel = np.linalg.norm(got - expect) / np.linalg.norm(expect)
    assert rel <= 2e-2, rel


def test_full_size_layer_exit_one_sequence_vs_oracle(gpu_lib):
    """13b_layer (Llama-2 13B Layer exit: 40 heads, F 13824, V 32000) at the
    bench's full 16 x 2048 tokens, one exit = the launches bench.py repeats
    per exit.  The oracle runs the exit forward on one whole sequence (the
    last, 2048 tokens: attention couples a sequence's rows) and every row of it
    is compared (lse, loss_t, confidence, argmax under A9); loss = mean of the
    per-token losses; P4 on dW_out; finite gradients; bitwise determinism."""
    from harness import attn_kwargs
    ee = gpu_lib
    cfg = _one_exit("13b_layer")
    n, T = cfg.tokens, cfg.seq_len
    hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
    targets = S.targets(cfg, n, device="cuda")
    params = S.head_params(cfg, device="cuda")
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, "layer", **attn_kwargs(cfg))
    ops = [{k: (v.float().contiguous() if k.startswith("g_") else v.to(torch.bfloat16).contiguous())
            for k, v in params[0].items()}]

    def run():
        grads = [{k: torch.empty(v.shape, device="cuda") for k, v in params[0].items()}]
        ax = [{"lse": torch.zeros(n, device="cuda"), "loss_tok": torch.zeros(n, device="cuda"),
               "argmax": torch.zeros(n, dtype=torch.int32, device="cuda"),
               "conf": torch.zeros(n, device="cuda")}]
        ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
        loss = torch.zeros(1, device="cuda")
        ee.ee_tune_step(c, hidden, targets, [1.0], ops, grads, loss, ws, aux=ax)
        torch.cuda.synchronize()
        return loss, grads, ax, ee.ee_get_status(ws)

    loss, grads, aux, st = run()
    assert st == (0, -1)
    seq = slice(n - T, n)
    p64 = {k: to_f64(v) for k, v in ops[0].items()}
    act = O.exit_forward("layer", p64, to_f64(hidden[0][seq]), 1e-5, S.attn_geometry(cfg))
    tg = targets.cpu().numpy()
    st_o = O.lm_loss_stats(act["S"], tg[seq])
    lse = aux[0]["lse"].cpu().numpy()[seq]
    assert np.max(np.abs(lse - st_o["lse"])) <= 5e-2
    assert np.max(np.abs(aux[0]["conf"].cpu().numpy()[seq] - st_o["conf"])) <= 2e-2
    lt = aux[0]["loss_tok"].cpu().numpy()[seq]
    assert np.max(np.abs(lt - st_o["loss"])) <= 5e-2
    assert abs(lt.mean() - st_o["loss"].mean()) <= 1e-3 * st_o["loss"].mean()
    check_argmax(aux[0]["argmax"].cpu().numpy()[seq], act["S"])
    valid = tg != -1
    lt_all = aux[0]["loss_tok"].double().cpu().numpy()
    assert abs(loss.item() - lt_all[valid].mean()) <= 1e-5 * abs(loss.item())
    dw = grads[0]["w_out"].double()
    assert dw.sum(dim=0).norm().item() <= 1e-2 * dw.abs().sum(dim=0).norm().item()
    for k, g in grads[0].items():
        assert torch.isfinite(g).all(), k
        assert g.abs().sum().item() > 0, k
    loss2, grads2, _, _ = run()
    assert torch.equal(loss, loss2)
    for k in grads[0]:
        assert torch.equal(grads[0][k], grads2[0][k]), k


@pytest.mark.parametrize("name", ["70b", "13b"])
def test_full_size_long_k_equals_sum_of_short_k_shards(gpu_lib, name):
    """P10 (linearity over tokens, P:183-188 + A16) at the bench's full size:
    the step on all N tokens -- weight-gradient GEMMs with K = N >= 16384 on
    the static wave-barrier schedule over thousands of pair tiles -- equals
    the sum of the steps on N/8-token shards (K = 8192: the dynamic tile
    schedule, a different code path) accumulated with the global valid count,
    to fp32 summation-order tolerance on every gradient tensor.  The shard
    path is itself pinned to the oracle (test_gpu_parity, test_gpu_largen)."""
    ee = gpu_lib
    cfg = _one_exit(name)
    n = cfg.tokens
    hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
    targets = S.targets(cfg, n, device="cuda")
    params = S.head_params(cfg, device="cuda")
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, cfg.arch)
    ops = [{k: (v.float().contiguous() if k.startswith("g_") else v.to(torch.bfloat16).contiguous())
            for k, v in params[0].items()}]
    del params
    ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
    full = [{k: torch.empty(v.shape, device="cuda") for k, v in ops[0].items()}]
    loss_full = torch.zeros(1, device="cuda")
    ee.ee_tune_step(c, hidden, targets, [1.0], ops, full, loss_full, ws)
    W = torch.zeros(1, dtype=torch.int64, device="cuda")
    ee.ee_count_valid(targets, cfg.vocab, W, ws)
    shard = [{k: torch.empty(v.shape, device="cuda") for k, v in ops[0].items()}]
    loss_sum, loss_s = 0.0, torch.zeros(1, device="cuda")
    m = n // 8
    for s in range(8):
        ee.ee_tune_step(c, [hidden[0][s * m:(s + 1) * m]], targets[s * m:(s + 1) * m], [1.0], ops,
                        shard, loss_s, ws, accumulate=s > 0, valid_count=W)
        loss_sum += loss_s.item()
    torch.cuda.synchronize()
    assert ee.ee_get_status(ws) == (0, -1)
    assert abs(loss_full.item() - loss_sum) <= 1e-5 * loss_full.item()
    errs = {}
    for k in full[0]:
        a, b = full[0][k].double(), shard[0][k].double()
        errs[k] = ((a - b).norm() / b.norm()).item()
        assert errs[k] <= 3e-4, (k, errs[k])
    print(name, {k: f"{e:.1e}" for k, e in errs.items()})


def test_full_size_bench_path_equals_plain_step(gpu_lib):
    """The bench's launch configuration at full size (70B head, 65 536 tokens,
    the fused ZeRO-1 path at world 1: gradient rows stored by the scatter
    epilogues into the arena, peer barrier, sharded Adam storing the operands)
    gives bitwise the losses and updated parameters of the plain path
    (ee_tune_step + ee_adam_update), which the tests above pin to the oracle."""
    from paper_2402_00518_b200.parallel import ShardedDPHeads
    ee = gpu_lib
    cfg = _one_exit("70b")
    n = cfg.tokens
    spec = ee.HeadSpec(cfg.hidden, cfg.vocab, cfg.ffn, 1, cfg.arch)
    src = [{k: v for k, v in S.head_params(cfg, device="cuda")[0].items()}]
    hidden = [h.contiguous() for h in S.hidden_states(cfg, n, device="cuda")]
    targets = S.targets(cfg, n, device="cuda")
    plain = ee.ExitHeads(spec, n)
    plain.init("copy", copy_src=src, src_dtype=torch.float32)
    lp = plain.step(hidden, targets).clone()
    plain.adam(1e-4)
    torch.cuda.synchronize()
    ops = {k: v.clone() for k, v in plain.operand[0].items()}
    del plain
    torch.cuda.empty_cache()
    heads = ShardedDPHeads(spec, n, 0, 1)
    heads.connect_local([heads])
    heads.init("copy", copy_src=src, src_dtype=torch.float32)
    ls = heads.step(hidden, targets, 1e-4).clone()
    torch.cuda.synchronize()
    assert heads.status() == (0, -1)
    assert torch.equal(lp, ls), (lp, ls)
    for k, v in ops.items():
        assert torch.equal(heads.operand[0][k], v), k
