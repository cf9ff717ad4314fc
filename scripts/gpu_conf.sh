timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -k confident -p no:cacheprovider > gpurun_out/pytest_conf_r01f.log 2>&1; echo "rc=$?"
grep -E "^(64|256)|passed|failed|^E " gpurun_out/pytest_conf_r01f.log | head
