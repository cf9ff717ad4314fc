"""Confidence-based early-exit decision (NEXT #4) on the GPU vs the
fp64 oracle: greedy token (argmax, gap rule A9), confidence, first exit."""

import numpy as np
import pytest
import torch

import eesynth as S
from eesynth import to_f64
from harness import check_argmax
from oracle import ee_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch,h,V,F,n", [("mlp", 256, 4104, 512, 300), ("norm", 128, 1000, 0, 8),
                                          ("embedding", 192, 2056, 0, 77),
                                          # decode shapes (n <= 16): the skinny weight-streaming path
                                          ("mlp", 256, 4104, 512, 1), ("mlp", 384, 1000, 640, 8),
                                          ("mlp", 256, 2056, 384, 13), ("norm", 128, 1000, 0, 16),
                                          ("embedding", 192, 2056, 0, 3), ("norm", 128, 1000, 0, 5)])
def test_exit_infer_matches_oracle(gpu_lib, arch, h, V, F, n):
    ee = gpu_lib
    cfg = S.Cfg(name="small", hidden=h, vocab=V, ffn=F, arch=arch, tokens=n, layers=3,
                after=[1, 2, 3], init="random", seed=31)
    hidden = S.hidden_states(cfg, n)
    params = S.head_params(cfg)
    c = ee.make_config(h, V, F, 3, arch)
    ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().to(torch.bfloat16))
            for k, v in p.items()} for p in params]
    am = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(3)]
    cf = [torch.zeros(n, device="cuda") for _ in range(3)]
    first = torch.zeros(n, dtype=torch.int32, device="cuda")
    ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
    p64 = [{k: to_f64(v) for k, v in p.items()} for p in params]
    _, cf_o, _ = O.exit_infer(arch, p64, [to_f64(x) for x in hidden], 1.0, 1e-5)
    tau = float(np.median(cf_o))
    ee.ee_exit_infer(c, [x.cuda() for x in hidden], ops, tau, am, cf, ws, first_exit=first)
    torch.cuda.synchronize()
    am_o, cf_o, first_o = O.exit_infer(arch, p64, [to_f64(x) for x in hidden], tau, 1e-5)
    for i in range(3):
        S_i = O.exit_forward(arch, p64[i], to_f64(hidden[i]), 1e-5)["S"]
        check_argmax(am[i].cpu().numpy(), S_i)
        assert np.max(np.abs(cf[i].cpu().numpy() - cf_o[i])) <= 2e-2
    fg = first.cpu().numpy()
    cfg_np = np.array([c_.cpu().numpy() for c_ in cf])
    for t in range(n):   # exact except where an exit's confidence sits within 1e-3 of tau
        near = np.any(np.abs(cf_o[:, t] - tau) < 1e-3)
        if not near:
            assert fg[t] == first_o[t], t
        expect_gpu = next((i for i in range(3) if cfg_np[i, t] >= tau), -1)
        assert fg[t] == expect_gpu


@pytest.mark.parametrize("arch,h,V,F,n", [("mlp", 2048, 8008, 5760, 1), ("mlp", 2048, 8008, 5760, 16),
                                          ("mlp", 1088, 4104, 2944, 11), ("norm", 4096, 32000, 0, 8),
                                          ("embedding", 4096, 32000, 0, 2)])
def test_exit_infer_decode_stream_k(gpu_lib, arch, h, V, F, n):
    """Decode shapes whose (row block, k chunk) units outnumber the CTAs, so the
    stream-K ranges split row blocks between CTAs (skinny.cu fix-up pool; K
    tails: F = 5760, 2944 and h = 1088 are not multiples of the 256-wide k chunk):
    oracle parity, and two calls bitwise equal."""
    ee = gpu_lib
    E = 2
    cfg = S.Cfg(name="dec", hidden=h, vocab=V, ffn=F, arch=arch, tokens=n, layers=E,
                after=list(range(1, E + 1)), init="random", seed=77)
    hidden = S.hidden_states(cfg, n)
    params = S.head_params(cfg)
    c = ee.make_config(h, V, F, E, arch)
    ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().to(torch.bfloat16))
            for k, v in p.items()} for p in params]
    ws = torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
    p64 = [{k: to_f64(v) for k, v in p.items()} for p in params]
    outs = []
    for _ in range(2):
        am = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(E)]
        cf = [torch.zeros(n, device="cuda") for _ in range(E)]
        first = torch.zeros(n, dtype=torch.int32, device="cuda")
        ee.ee_exit_infer(c, [x.cuda() for x in hidden], ops, 0.5, am, cf, ws, first_exit=first)
        torch.cuda.synchronize()
        outs.append((am, cf, first))
    for i in range(E):
        assert torch.equal(outs[0][0][i], outs[1][0][i]) and torch.equal(outs[0][1][i], outs[1][1][i])
    assert torch.equal(outs[0][2], outs[1][2])
    am, cf, _ = outs[0]
    _, cf_o, _ = O.exit_infer(arch, p64, [to_f64(x) for x in hidden], 0.5, 1e-5)
    for i in range(E):
        S_i = O.exit_forward(arch, p64[i], to_f64(hidden[i]), 1e-5)["S"]
        check_argmax(am[i].cpu().numpy(), S_i)
        assert np.max(np.abs(cf[i].cpu().numpy() - cf_o[i])) <= 2e-2


def test_exit_infer_decode_concurrent_streams(gpu_lib):
    """Decode calls executing concurrently on several streams (each with its own
    workspace) share the library's stream-K fix-up pool by slot: every stream's
    results equal its serial run bitwise (include/ee.h: up to 16 concurrently
    executing calls)."""
    ee = gpu_lib
    h, V, F, E, n = 2048, 8008, 5760, 2, 3
    cfg = S.Cfg(name="dec", hidden=h, vocab=V, ffn=F, arch="mlp", tokens=n, layers=E,
                after=[1, 2], init="random", seed=91)
    params = S.head_params(cfg)
    c = ee.make_config(h, V, F, E, "mlp")
    ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().to(torch.bfloat16))
            for k, v in p.items()} for p in params]
    nstreams = 6
    inputs = [[x.cuda() for x in S.hidden_states(cfg, n, seed=200 + s)] for s in range(nstreams)]
    ws = [torch.zeros(ee.ee_workspace_size(c, n), dtype=torch.uint8, device="cuda")
          for _ in range(nstreams)]

    def outs():
        return ([torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(E)],
                [torch.zeros(n, device="cuda") for _ in range(E)])
    serial = []
    for s in range(nstreams):
        am, cf = outs()
        ee.ee_exit_infer(c, inputs[s], ops, 0.5, am, cf, ws[s])
        torch.cuda.synchronize()
        serial.append((am, cf))
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    conc = [outs() for _ in range(nstreams)]
    torch.cuda.synchronize()
    for rep in range(3):
        for s in range(nstreams):
            with torch.cuda.stream(streams[s]):
                ee.ee_exit_infer(c, inputs[s], ops, 0.5, conc[s][0], conc[s][1], ws[s],
                                 stream=streams[s])
        torch.cuda.synchronize()
        for s in range(nstreams):
            for i in range(E):
                assert torch.equal(conc[s][0][i], serial[s][0][i]), (rep, s, i)
                assert torch.equal(conc[s][1][i], serial[s][1][i]), (rep, s, i)
