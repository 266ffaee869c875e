# r02ay: same-box A/B of the parameter-upload threshold (C2, C3), interleaved
set -x
T=r02ay
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for rep in 1 2 3; do
for prm in 0 4096 31744; do
  for c in C2 C3; do
  GVOX_H2D_PARAM=$prm timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --per-call-runs 20 --e2e-steps 40 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c param=$prm', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4))" >> gpurun_out/${T}_configs.log
  done
done
done
ls -la gpurun_out | grep ${T}
