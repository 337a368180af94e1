#!/usr/bin/env bash
# A/B: cooperative CSR window (default build) vs per-batch broadcast loads (csr0), PA MINB 5
OUT=gpurun_out/ab_csr; mkdir -p $OUT
L=paper_2501_19221_b200/_lib
for rep in 1 2; do
for v in csr0 main csr1m5; do
  if [ $v = main ]; then lib=$L/libvxq.so; else lib=$L/libvxq_$v.so; fi
  for a in "cfg3 pa" "cfg4 pa" "cfg3 sbm" "cfg4 sbm" "cfg5 pa"; do
    set -- $a
    extra=""; [ $1 = cfg5 ] && extra="--steps 2 --warmup 1"
    VXQ_LIB=$lib timeout 600 python bench.py --config $1 --solver $2 --steps 4 --warmup 3 --no-cpu --no-e2e $extra > $OUT/${v}_$1_$2_$rep.json 2> $OUT/${v}_$1_$2_$rep.err
    python -c "import json;d=json.loads(open('$OUT/${v}_$1_$2_$rep.json').read().splitlines()[-1]);print('$v $1 $2', round(d['roofline']['mean_launch_ms']*1000,1),'us', round(d['roofline']['frac'],3))" 2>/dev/null || echo "$v $1 $2 FAILED"
  done
done
done
