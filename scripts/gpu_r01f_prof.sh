TAG=${1:-r01f}
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k confident -s > gpurun_out/pytest_conf_$TAG.log 2>&1; echo "conf rc=$?"; tail -5 gpurun_out/pytest_conf_$TAG.log
timeout 1500 bash scripts/gpu_ncu.sh $TAG; echo "ncu rc=$?"
