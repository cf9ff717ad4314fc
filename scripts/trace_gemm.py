"""Per-tile timing trace of one big GEMM (debug): how far apart in time do the
CTAs sharing an operand block reach the same k-range?  Prints wave spreads."""
import ctypes, os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00518_b200 as ee

lib = ee.load()
lib.ee_debug_trace_read.restype = ctypes.c_int32
lib.ee_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int32]
M, N, K = 65536, 28672, 8192
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda")
ee.ee_test_gemm(A, B, C, True, True, M, N, K)
torch.cuda.synchronize()
lib.ee_debug_trace_arm()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ee.ee_test_gemm(A, B, C, True, True, M, N, K)
e1.record()
torch.cuda.synchronize()
n = 1 << 20
buf = (ctypes.c_uint64 * n)()
got = lib.ee_debug_trace_read(buf, n)
t = [buf[i] >> 8 for i in range(got)]
sm = [buf[i] & 0xFF for i in range(got)]
cta2 = os.environ.get("EE_GEMM_CTA", "1") == "2"
P = 74 if cta2 else 148
t0 = min(t)
dur = e0.elapsed_time(e1)
print(f"mode cta2={cta2} cluster={os.environ.get('EE_GEMM_CLUSTER','1')} tiles={got} ms={dur:.2f}")
waves = [t[i:i + P] for i in range(0, got, P)]
per_tile = dur * 1e6 / (got / P)
spreads = [(max(w) - min(w)) / per_tile for w in waves if len(w) == P]
print("wave spread / tile time: first", [round(x, 2) for x in spreads[:5]], "median",
      round(statistics.median(spreads), 2), "max", round(max(spreads), 2))
# tiles of wave 100: sorted by SM id, show start offsets
w = 100
idx = list(range(w * P, (w + 1) * P))
print("wave", w, "offsets(us) by tile order:", [round((t[i] - min(t[j] for j in idx)) / 1e3, 1) for i in idx[:40]])
print("smids:", [sm[i] for i in idx[:40]])
