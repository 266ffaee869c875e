# r02bf: host laps of the C5 build (GVOX_DEBUG_TIMING) in the timed step
set -x
T=r02bf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
GVOX_DEBUG_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
ls -la gpurun_out | grep ${T}
