#!/usr/bin/env bash
# A/B: packed FADD2/FMUL2 accumulation in the sparse step kernels (main) vs scalar (f2off)
OUT=gpurun_out/ab_f2; mkdir -p $OUT
L=paper_2501_19221_b200/_lib
for rep in 1 2; do
for v in f2off main; do
  if [ $v = main ]; then lib=$L/libvxq.so; else lib=$L/libvxq_$v.so; fi
  for a in "cfg3 pa" "cfg4 pa" "cfg3 sbm" "cfg4 sbm"; do
    set -- $a
    VXQ_LIB=$lib timeout 600 python bench.py --config $1 --solver $2 --steps 4 --warmup 3 --no-cpu --no-e2e > $OUT/${v}_$1_$2_$rep.json 2> $OUT/${v}_$1_$2_$rep.err
    python -c "import json;d=json.loads(open('$OUT/${v}_$1_$2_$rep.json').read().splitlines()[-1]);print('$v $1 $2', round(d['roofline']['mean_launch_ms']*1000,1),'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || echo "$v $1 $2 FAILED"
  done
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
