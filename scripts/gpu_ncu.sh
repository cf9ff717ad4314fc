#!/bin/bash
# ncu evidence for bench.py's default step (one GPU; never under torchrun):
# the launch list of one step (cold-cache, serialised) and --set full captures
# of one exit's GEMMs and of the bandwidth kernels.  Reports are summarised on
# the CPU side with scripts/ncu_summary.py.
TAG=${1:-r02}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -s 0 -c 10 \
    -o gpurun_out/prof_gemm_$TAG python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rmsnorm|adam|gain_grad|ce_finalize|transpose|reduce_cols" -s 0 -c 12 \
    -o gpurun_out/prof_bw_$TAG python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_bw_$TAG.log 2>&1
ls -la gpurun_out/ | tail -8
