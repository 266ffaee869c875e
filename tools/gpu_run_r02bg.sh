# r02bg: GPU-side phase times of the C5 e2e step (events, no syncs)
set -x
T=r02bg
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
GVOX_E2E_EVENTS=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 10 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
GVOX_DEBUG_TIMING=1 GVOX_E2E_EVENTS=1 timeout 300 python bench.py --config C2 --steps 20 --no-cpu-baseline --per-call-runs 0 --e2e-steps 20 > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
ls -la gpurun_out | grep ${T}
