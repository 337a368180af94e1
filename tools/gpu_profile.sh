#!/usr/bin/env bash
# Round profiling recipe (run on the GPU box via gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh <tag>'
# 1. GPU parity suite, 2. bench lines (cfg2/cfg4/cfg5), 3. ncu launch list of the
# default bench command, 4. one `ncu --set full` capture per top kernel.
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NCU=${NCU:-ncu}

timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" | tee -a "$OUT/status.txt"

timeout 600 python bench.py > "$OUT/bench_cfg2.json" 2> "$OUT/bench_cfg2.err"
echo "bench cfg2 rc=$?" | tee -a "$OUT/status.txt"
timeout 600 python bench.py --config cfg4 > "$OUT/bench_cfg4.json" 2> "$OUT/bench_cfg4.err"
echo "bench cfg4 rc=$?" | tee -a "$OUT/status.txt"
timeout 900 python bench.py --config cfg5 --steps 3 > "$OUT/bench_cfg5.json" 2> "$OUT/bench_cfg5.err"
echo "bench cfg5 rc=$?" | tee -a "$OUT/status.txt"

# launch list of the default bench command (cold-cache, serialised per-launch times)
if timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; then
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches_bench_cfg2.csv" python bench.py --steps 1 --warmup 3 --no-cpu \
    > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?" | tee -a "$OUT/status.txt"
fi

cap() {  # cap <name> <kernel regex> <profile_run args...>
  local name=$1 kern=$2; shift 2
  if timeout 300 python tools/profile_run.py "$@" > "$OUT/plain_$name.log" 2>&1; then
    VXQ_WAIT_TIMEOUT_S=600 VXQ_DENSE_NOCOOP=1 timeout 900 $NCU --set full --clock-control none --import-source on \
      -k "regex:$kern" -s 2 -c 1 -o "$OUT/$name" -f python tools/profile_run.py "$@" \
      > "$OUT/ncu_$name.log" 2>&1
    echo "ncu $name rc=$?" | tee -a "$OUT/status.txt"
  else
    echo "plain $name failed" | tee -a "$OUT/status.txt"
  fi
}
cap dense_cfg2 k_dense_run --config cfg2 --T 8
cap sparse_cfg4 k_pa_step --config cfg4 --T 8
cap coop_cfg5 k_pa_step_coop --config cfg5 --T 4 --repeat 1
cap sbm_cfg4 k_sbm_step --config cfg4 --T 8 --solver sbm
echo done
