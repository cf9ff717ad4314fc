TAG=${1:-r01f}
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu_$TAG.log
grep -E "^(64|256)\.0 " gpurun_out/pytest_gpu_$TAG.log | head
python - <<'PY'
import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory(); y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); [y.copy_(x, non_blocking=True) for _ in range(5)]; e1.record(); torch.cuda.synchronize()
print("H2D pinned GB/s", 5 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9)
PY
