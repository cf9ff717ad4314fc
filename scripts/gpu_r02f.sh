#!/bin/bash
# r02f: full-size long-K vs shard-sum test, strong-scaling DP rank emulation,
# compute-sanitizer memcheck of the comm kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rA -k long_k > gpurun_out/r02f_fullsize.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_fullsize.log
for P in 1 2 4 8; do
  timeout 600 python scripts/dp_emulate.py --config 70b_dp --ranks $P --strong >> gpurun_out/r02f_dp_emulate_strong.jsonl 2>>gpurun_out/r02f_dp_emulate.err
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_comm.py -q -x -k "mlp-2 or embedding or two_processes" > gpurun_out/r02f_memcheck_comm.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_memcheck_comm.log
tail -3 gpurun_out/r02f_fullsize.log; cat gpurun_out/r02f_dp_emulate_strong.jsonl | cut -c1-300; tail -5 gpurun_out/r02f_memcheck_comm.log
timeout 600 python bench.py --config 70b --parallel vp --no-cpu-baseline --no-ds-ablation > gpurun_out/r02f_bench_vp70_n1.json 2> gpurun_out/r02f_bench_vp.err
timeout 600 python bench.py --gpus 2 --config 13b --parallel vp --steps 3 --no-e2e > gpurun_out/r02f_bench_vp13_2ranks.json 2>> gpurun_out/r02f_bench_vp.err
timeout 600 python bench.py --config 70b --dp-comm plain --no-cpu-baseline > gpurun_out/r02f_bench_c3_70b.json 2>> gpurun_out/r02f_bench_vp.err
cut -c1-400 gpurun_out/r02f_bench_vp70_n1.json gpurun_out/r02f_bench_vp13_2ranks.json gpurun_out/r02f_bench_c3_70b.json
