timeout 900 python bench.py --parallel vp --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d.pop('kernels'); print(json.dumps(d)); print({n: round(v['ms_per_launch'],2) for n,v in k.items()})"
EE_GEMM_CTA=2 ncu --set full --clock-control none -k regex:gemm -s 0 -c 3 -o gpurun_out/prof_cta2 python bench.py --quick --steps 1 --warmup 0 > gpurun_out/ncu_cta2.log 2>&1
tail -3 gpurun_out/ncu_cta2.log
