# r02h: recycled dense grids (no per-build fill), pinned build metadata upload:
# GPU tests, C5 bench line, small-config steps.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02h_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; print('$c', 'step', round(d['ms_per_step'],4), 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'host', {k: round(v,4) for k,v in s['host_wall_ms_per_step'].items()})" >> gpurun_out/r02h_configs.log
done
GVOX_DEBUG_TIMING=1 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > /dev/null 2> gpurun_out/r02h_c2_build_laps.log
