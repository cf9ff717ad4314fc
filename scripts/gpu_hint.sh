M="--metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control base -k regex:gemm -s 0 -c 3"
for cfg in "2 -1 -1" "2 1 1" "2 2 1" "2 1 2" "1 1 1" "1 2 1" "1 1 2"; do
set -- $cfg
echo "CTA=$1 HINT_A=$2 HINT_B=$3"
EE_GEMM_CTA=$1 EE_GEMM_HINT_A=$2 EE_GEMM_HINT_B=$3 ncu $M python bench.py --quick --steps 1 --warmup 0 2>&1 | grep -E "dram__bytes|duration|hit_rate" | awk '{printf "%s %s  ", $1, $3} END {print ""}'
done
