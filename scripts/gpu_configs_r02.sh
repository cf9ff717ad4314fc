#!/bin/bash
# r02 config sweep on one box: default C4 line, C3 (70b), C2 (13b), C1 (7b), 13b_layer.
TAG=${1:-r02n}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}.err
for c in 70b 13b 7b 13b_layer; do
  timeout 900 python bench.py --config $c --dp-comm plain --no-cpu-baseline > gpurun_out/${TAG}_$c.json 2>> gpurun_out/${TAG}.err
done
for f in gpurun_out/${TAG}_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['ms_per_step'],1), round(d['pct_peak']['of_burst'],4), d['clocks']['sm_mhz'], (d.get('ds_ablation') or {}).get('value'), (d.get('e2e') or {}).get('value'), d['roofline']['kernel'], round(d['roofline']['frac'],3))"; done
for c in 13b_q 70b_q; do
  timeout 900 python bench.py --parallel pp --config $c --steps 3 > gpurun_out/${TAG}_pp_$c.json 2>> gpurun_out/${TAG}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_pp_$c.json').read().strip().splitlines()[-1])
print('pp $c', round(d['value']), round(d['ms_per_step'],1), round(d['pct_peak']['of_burst'],4), d['clocks']['sm_mhz'])"
done
