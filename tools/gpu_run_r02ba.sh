# r02ba: no pinned-slot event for blocks uploaded as launch parameters;
# GPU suite; C1-C3 (3 x C2)
set -x
T=r02ba
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for c in C2 C1 C3 C2 C2; do
  timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --per-call-runs 20 --e2e-steps 40 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4))" >> gpurun_out/${T}_configs.log
done
ls -la gpurun_out | grep ${T}
