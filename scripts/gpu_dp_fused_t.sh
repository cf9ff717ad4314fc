TAG=${1:-r01f}
timeout 900 python -m pytest tests/test_gpu_dp_fused.py tests/test_gpu_vp_fused.py -x -q > gpurun_out/pytest_dpfused_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_dpfused_$TAG.log
