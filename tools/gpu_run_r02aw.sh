# r02aw: every small input block (multi-segment uploads included) in the
# launch parameters by default; GPU suite; C1-C3 step / e2e; C5 bench line
set -x
T=r02aw
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for c in C1 C2 C3 C2; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4))" >> gpurun_out/${T}_configs.log
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --per-call-runs 5 --e2e-steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'per_call', round(d['per_call']['ms_median'],3))" >> gpurun_out/${T}_configs.log
ls -la gpurun_out | grep ${T}
