# r02j: sync-free small builds, pinned staging ring, device-resident counts in
# the small-config step: GPU tests, C5 bench, config table, ncu of k_linearize.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02j_pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; print('$c', 'step', round(d['ms_per_step'],4), 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'host', {k: round(v,4) for k,v in s['host_wall_ms_per_step'].items()})" >> gpurun_out/r02j_configs.log
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o gpurun_out/r02j_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/r02j_ncu_lin.log 2>&1
