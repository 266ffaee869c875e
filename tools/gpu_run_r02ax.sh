# r02ax: input blocks up to 4 KB in the launch parameters (default); C1-C3
set -x
T=r02ax
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${T}_pytest_parity.log 2>&1
for c in C1 C2 C3 C2 C1; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4))" >> gpurun_out/${T}_configs.log
done
ls -la gpurun_out | grep ${T}
