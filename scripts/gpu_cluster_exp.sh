M="--metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control base -k regex:gemm -s 0 -c 3"
for cl in 1 2; do
echo "CTA=1 CLUSTER=$cl"
EE_GEMM_CLUSTER=$cl ncu $M python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "dram__bytes|duration|hit_rate" | awk '{printf "%s %s  ", $1, $3} END {print ""}'
done
