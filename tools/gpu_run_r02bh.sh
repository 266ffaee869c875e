# r02bh: C5 e2e with the next step's upload issued after the screened batch's
# launch vs at the step start (A/B x2), phase events
set -x
T=r02bh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for m in late early late early; do
  if [ $m = early ]; then export GVOX_E2E_EARLY_UPLOAD=1; else unset GVOX_E2E_EARLY_UPLOAD; fi
  GVOX_E2E_EVENTS=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 20 > gpurun_out/${T}_bench_$m.json 2> gpurun_out/${T}_bench_$m.err
  python -c "import json; d=json.loads(open('gpurun_out/${T}_bench_$m.json').read().strip().splitlines()[-1]); print('$m', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))" >> gpurun_out/${T}_e2e.log
  grep "e2e events" gpurun_out/${T}_bench_$m.err >> gpurun_out/${T}_e2e.log
done
timeout 300 python bench.py --config C2 --steps 50 --no-cpu-baseline --per-call-runs 0 --e2e-steps 40 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))" >> gpurun_out/${T}_e2e.log
ls -la gpurun_out | grep ${T}
