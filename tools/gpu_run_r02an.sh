# r02an: e2e A/B -- result readback on a D2H stream vs synchronous (C5)
set -x
T=r02an
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for m in async sync async; do
  if [ $m = sync ]; then export GVOX_E2E_SYNC_READBACK=1; else unset GVOX_E2E_SYNC_READBACK; fi
  GVOX_E2E_DEBUG=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 10 > gpurun_out/${T}_bench_$m.json 2> gpurun_out/${T}_bench_$m.err
done
ls -la gpurun_out | grep ${T}
