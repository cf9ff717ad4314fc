# compute-sanitizer on the tiny config and small ragged shapes (SURVEY test tier 6)
for tool in memcheck synccheck; do
echo "== $tool"
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or small_ragged" 2>&1 | tail -8
done
echo "== memcheck 1-CTA kernel"
EE_GEMM_CTA=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny" 2>&1 | tail -4
