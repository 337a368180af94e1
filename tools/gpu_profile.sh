#!/usr/bin/env bash
# Round evidence recipe (run on the GPU box via gpurun from the repo root):
#   gpurun --timeout 3600 -- 'bash tools/gpu_profile.sh <tag>'
# 1. GPU parity suite + smoke, 2. bench lines (every config / solver, the reference arm),
# 3. ncu launch list of the default bench command, 4. one `ncu --set full` capture per top
# kernel.  Each ncu command runs only after the same command exited 0 without ncu.
# Summaries: python tools/ncu_summary.py gpurun_out/<tag>/*.ncu-rep gpurun_out/<tag>/*.csv
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NCU=${NCU:-ncu}
# persistent dense kernels wait on each other's tiles: ncu replays need a plain launch and
# a long spin-wait timeout
NCUENV="VXQ_DENSE_NOCOOP=1 VXQ_WAIT_TIMEOUT_S=600"

timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" | tee -a "$OUT/status.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" | tee -a "$OUT/status.txt"

timeout 600 python bench.py > "$OUT/bench_cfg2.json" 2> "$OUT/bench_cfg2.err"
echo "bench cfg2 rc=$?" | tee -a "$OUT/status.txt"
timeout 600 python bench.py --impl reference > "$OUT/bench_cfg2_reference.json" 2> "$OUT/ref.err"
echo "ref rc=$?" | tee -a "$OUT/status.txt"
for a in "cfg2 sbm" "cfg3 pa" "cfg3 sbm" "cfg4 pa" "cfg4 sbm"; do
  set -- $a
  timeout 600 python bench.py --config $1 --solver $2 > "$OUT/bench_$1_$2.json" 2> "$OUT/bench_$1_$2.err"
  echo "bench $1 $2 rc=$?" | tee -a "$OUT/status.txt"
done
timeout 900 python bench.py --config cfg5 --steps 3 --no-cpu > "$OUT/bench_cfg5_pa.json" 2> "$OUT/bench_cfg5.err"
echo "bench cfg5 rc=$?" | tee -a "$OUT/status.txt"
for s in pa sbm; do
  timeout 600 python bench.py --config cfg1 --nvars 10000 --replicas 1024 --solver $s \
    > "$OUT/bench_dense_general_$s.json" 2> "$OUT/bench_dg_$s.err"
  echo "bench general $s rc=$?" | tee -a "$OUT/status.txt"
done

# launch list of the default bench command (cold-cache, serialised per-launch times)
if timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; then
  env $NCUENV timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 \
    --csv --log-file "$OUT/launches_bench_cfg2.csv" python bench.py --steps 1 --warmup 3 \
    --no-cpu --no-e2e > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?" | tee -a "$OUT/status.txt"
fi

cap() {  # cap <name> <kernel regex> <skip> <profile_run args...>
  local name=$1 kern=$2 skip=$3; shift 3
  if timeout 300 python tools/profile_run.py "$@" > "$OUT/plain_$name.log" 2>&1; then
    env $NCUENV timeout 900 $NCU --set full --clock-control none --import-source on \
      -k "regex:$kern" -s "$skip" -c 1 -o "$OUT/$name" -f python tools/profile_run.py "$@" \
      > "$OUT/ncu_$name.log" 2>&1
    echo "ncu $name rc=$?" | tee -a "$OUT/status.txt"
  else
    echo "plain $name failed" | tee -a "$OUT/status.txt"
  fi
}
# dense solves launch the dynamics kernel then the energy pass: -s 2 = second solve's loop
cap dense_pa_cfg2 k_dense_run 2 --config cfg2 --T 8
cap dense_sbm_cfg2 k_dense_run 2 --config cfg2 --T 8 --solver sbm
cap dense_general_pa k_dense_run 1 --config cfg1 --n 10000 --replicas 1024 --T 8
cap sparse_cfg4 k_pa_step 2 --config cfg4 --T 8
cap sparse_cfg3 k_pa_step 2 --config cfg3 --T 8
cap sbm_cfg4 k_sbm_step 2 --config cfg4 --T 8 --solver sbm
cap coop_cfg5 k_pa_step_coop 1 --config cfg5 --T 4 --repeat 1
echo done
