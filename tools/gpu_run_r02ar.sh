# r02ar: recycled record arenas (small builds) and reused grid-pool events;
# k-NN G = 8 for single frames; GPU suite; C1-C3 steps
set -x
T=r02ar
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for c in C1 C2 C3 C2 C1 C2; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; h=s['host_wall_ms_per_step']; print('$c', 'step', round(d['ms_per_step'],4), 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'host', {k: round(v,4) for k,v in h.items()})" >> gpurun_out/${T}_configs.log
done
timeout 300 python tools/bench_preprocess.py > gpurun_out/${T}_bench_pre.json 2>/dev/null
ls -la gpurun_out | grep ${T}
