# r02au: e2e with one contiguous upload and the C1-C3 overlap counts kept on
# the device; C1-C3 and C5
set -x
T=r02au
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for c in C1 C2 C3 C2; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'h2d', d['e2e']['h2d_bytes_per_step'], 'd2h', d['e2e']['d2h_bytes_per_step'])" >> gpurun_out/${T}_configs.log
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --per-call-runs 3 --e2e-steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))" >> gpurun_out/${T}_configs.log
ls -la gpurun_out | grep ${T}
