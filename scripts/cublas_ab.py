"""Our tcgen05 GEMM (ee_test_gemm: fp32 output) against cuBLAS (torch.mm,
bf16 output) on the step's GEMM shapes at the 70B head shape, each timed for
~3 s sustained (the power-capped regime of the step), alternating the two
implementations on one box.  TFLOP/s = 2 M N K / time."""
import json, os, sys, subprocess, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2402_00518_b200 as ee
ee.load()
dev = torch.device("cuda")
N_TOK, h, F, V = 65536, 8192, 28672, 32000
SHAPES = [  # name, M, N, K, a_kmajor, b_kmajor
    ("8192^3", 8192, 8192, 8192, True, True),
    ("a2 [A|B] = u W^T", N_TOK, 2 * F, h, True, True),
    ("a5 S = z W_out^T", N_TOK, V, h, True, True),
    ("a12 dW = u^T [dA|dB]", h, 2 * F, N_TOK, True, False),
    ("a8 dz = dS W_out", N_TOK, h, V, True, False),
]


def smi():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                              capture_output=True, text=True).stdout.strip()
    except Exception:
        return ""


def timeit(fn, secs=3.0):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    one = e0.elapsed_time(e1)
    reps = max(2, int(secs * 1e3 / one))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    clk = smi()
    return e0.elapsed_time(e1) / reps, reps, clk


for name, M, N, K, ak, bk in SHAPES:
    g = torch.Generator(device=dev).manual_seed(1)
    A = (torch.randn(M, K, generator=g, device=dev) * 0.02).bfloat16() if ak else \
        (torch.randn(K, M, generator=g, device=dev) * 0.02).bfloat16()
    B = (torch.randn(N, K, generator=g, device=dev) * 0.02).bfloat16() if bk else \
        (torch.randn(K, N, generator=g, device=dev) * 0.02).bfloat16()
    C = torch.empty(M, N, device=dev)
    ours = lambda: ee.ee_test_gemm(A, B, C, ak, bk, M, N, K)
    At = A if ak else A.t()
    Bt = B.t() if bk else B
    Cb = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    cub = lambda: torch.mm(At, Bt, out=Cb)
    res = {"shape": name, "M": M, "N": N, "K": K}
    for tag, fn in (("ours_fp32_out", ours), ("cublas_bf16_out", cub), ("ours_fp32_out_2", ours),
                    ("cublas_bf16_out_2", cub)):
        ms, reps, clk = timeit(fn)
        res[tag] = {"ms": round(ms, 3), "tflops": round(2.0 * M * N * K / ms / 1e9, 1), "reps": reps,
                    "smi_clock_power_end": clk}
    print(json.dumps(res), flush=True)
    del A, B, C, Cb
    torch.cuda.empty_cache()
