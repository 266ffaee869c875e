# r02bd: per-kernel durations (ncu launch list) with and without the target
# execution order; and the candidate-sorted run for comparison
set -x
T=r02bd
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for eo in 1 0; do
  GVOX_LIN_EXEC_ORDER=$eo timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_eo$eo.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_ncu_eo$eo.log 2>&1
done
GVOX_LIN_EXEC_ORDER=0 GVOX_BENCH_PAIR_ORDER=target timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_sorted.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_ncu_sorted.log 2>&1
ls -la gpurun_out | grep ${T}
