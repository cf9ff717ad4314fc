TAG=${1:-r01f}
timeout 600 python -m pytest tests/test_gpu_adam_fused.py -x -q -p no:cacheprovider > gpurun_out/pytest_adamf_$TAG.log 2>&1; echo "pytest adamf rc=$?"
tail -15 gpurun_out/pytest_adamf_$TAG.log
