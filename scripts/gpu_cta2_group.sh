for g in 1 4 8 16 32; do
echo "GROUP=$g"
EE_GEMM_CTA=2 EE_GEMM_GROUP=$g ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -s 0 -c 3 python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "gemm2_kernel|dram__bytes|duration|hit_rate|per_second" | head -16
done
echo "CTA1 GROUP=16"
EE_GEMM_CTA=1 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -s 0 -c 3 python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "gemm_kernel|dram__bytes|duration|hit_rate|per_second" | head -16
