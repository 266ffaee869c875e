# r02bk: build metadata written straight into the pinned upload block;
# GPU suite, C5 step A/B against the previous state is not possible (no knob):
# laps + step
set -x
T=r02bk
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
GVOX_DEBUG_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_laps.json 2> gpurun_out/${T}_laps.err
for r in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --per-call-runs 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['stages'].items() if 'ms_per_step' in v and v['ms_per_step']}, d['clocks'])" >> gpurun_out/${T}_step.log; done
timeout 300 python bench.py --config C2 --steps 100 --no-cpu-baseline --per-call-runs 20 --e2e-steps 40 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))" >> gpurun_out/${T}_step.log
ls -la gpurun_out | grep ${T}
