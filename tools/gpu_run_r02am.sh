# r02am: e2e with the result readback on a D2H stream (C5 and C2)
set -x
T=r02am
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --per-call-runs 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 python bench.py --config C2 --steps 50 --no-cpu-baseline --per-call-runs 20 > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
ls -la gpurun_out | grep ${T}
