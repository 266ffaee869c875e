# r02ao: e2e A/B without debug syncs, 20 steps each, twice
set -x
T=r02ao
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for m in async sync async sync; do
  if [ $m = sync ]; then export GVOX_E2E_SYNC_READBACK=1; else unset GVOX_E2E_SYNC_READBACK; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))" >> gpurun_out/${T}_e2e.log
done
ls -la gpurun_out | grep ${T}
