set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --config 13b --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -3
