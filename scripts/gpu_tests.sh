nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(), torch.cuda.get_device_capability())"
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_init_optim.py -x -q 2>&1 | tail -40
