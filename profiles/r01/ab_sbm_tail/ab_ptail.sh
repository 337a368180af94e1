#!/usr/bin/env bash
# A/B: SBM step tail (1-3 entries) as one predicated batch (ptail) vs one-at-a-time (main)
OUT=gpurun_out/ab_ptail; mkdir -p $OUT
L=paper_2501_19221_b200/_lib
for rep in 1 2; do
for v in main ptail; do
  if [ $v = main ]; then lib=$L/libvxq.so; else lib=$L/libvxq_$v.so; fi
  for a in "cfg3 sbm" "cfg4 sbm" "cfg5 sbm"; do
    set -- $a
    extra=""; [ $1 = cfg5 ] && extra="--steps 2"
    VXQ_LIB=$lib timeout 600 python bench.py --config $1 --solver $2 --steps 4 --warmup 3 --no-cpu --no-e2e $extra > $OUT/${v}_$1_$2_$rep.json 2> $OUT/${v}_$1_$2_$rep.err
    python -c "import json;d=json.loads(open('$OUT/${v}_$1_$2_$rep.json').read().splitlines()[-1]);print('$v $1 $2', round(d['roofline']['mean_launch_ms']*1000,1),'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || echo "$v $1 $2 FAILED"
  done
done
done
VXQ_LIB=$L/libvxq_ptail.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
