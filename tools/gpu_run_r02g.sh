# r02g: incremental level bases on by default (GPU tests), occupancy variants
# of k_linearize, dense-ratio step sweep for the small configs, C2 build laps.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02g_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_pytest_gpu.log 2>&1
timeout 900 python tools/variants.py run base,lin_b5,lin_b6 > gpurun_out/r02g_variants_lin.log 2>&1
for r in 48 192 512 2048; do
  for c in C2 C3; do
    GVOX_DENSE_RATIO=$r timeout 300 python bench.py --config $c --steps 50 --no-e2e --no-cpu-baseline --per-call-runs 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; print('$r', '$c', 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'step', round(d['ms_per_step'],4), 'host', {k: round(v,4) for k,v in s['host_wall_ms_per_step'].items()})" >> gpurun_out/r02g_dense_sweep.log
  done
done
GVOX_DEBUG_TIMING=1 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > /dev/null 2> gpurun_out/r02g_c2_build_laps.log
