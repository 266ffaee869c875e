# r02bc: linearization tiles executed grouped by target map (device counting
# sort in the screened batch, host sort in gvox_linearize_batch); GPU suite;
# C5 A/B against the batch order
set -x
T=r02bc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for eo in 1 0 1 0; do
  GVOX_LIN_EXEC_ORDER=$eo timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('exec_order=$eo', round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['stages'].items() if 'ms_per_step' in v and v['ms_per_step']}, 'per_call', round(d['per_call']['ms_median'],2))" >> gpurun_out/${T}_ab.log
done
ls -la gpurun_out | grep ${T}
