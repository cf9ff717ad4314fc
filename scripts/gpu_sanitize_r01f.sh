for tool in memcheck synccheck; do
echo "== $tool"
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_r01f.py 2>&1 | tail -6
done
