# r02be: bench A/B of the target execution order, 20 steps, interleaved x3,
# with clocks; plus the candidate-sorted run
set -x
T=r02be
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for rep in 1 2 3; do
for eo in 1 0; do
  GVOX_LIN_EXEC_ORDER=$eo timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --per-call-runs 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('exec_order=$eo', round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['stages'].items() if 'ms_per_step' in v and v['ms_per_step']}, 'per_call', round(d['per_call']['ms_median'],2), d['clocks'])" >> gpurun_out/${T}_ab.log
done
done
ls -la gpurun_out | grep ${T}
