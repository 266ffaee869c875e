# r02as: C2 e2e laps (debug) and the plain C2 e2e
set -x
T=r02as
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
GVOX_E2E_DEBUG=1 timeout 300 python bench.py --config C2 --steps 20 --no-cpu-baseline --per-call-runs 0 --e2e-steps 10 > gpurun_out/${T}_c2_dbg.json 2> gpurun_out/${T}_c2_dbg.err
timeout 300 python bench.py --config C2 --steps 20 --no-cpu-baseline --per-call-runs 0 --e2e-mode serial > gpurun_out/${T}_c2_serial.json 2> gpurun_out/${T}_c2_serial.err
ls -la gpurun_out | grep ${T}
