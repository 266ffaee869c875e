# r02ad: fixes (selection-path tile map), counters zeroed by the insert
# descriptors' upload, counts copied by the finalize; the whole GPU suite;
# C1-C3 steps against the parameter-copy threshold; memcheck of the build path.
set -x
T=r02ad
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for c in C1 C2 C3; do
  for prm in 0 1024 4096 32000 4096; do
    GVOX_H2D_PARAM=$prm timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; h=s['host_wall_ms_per_step']; print('$c param=$prm', 'step', round(d['ms_per_step'],4), 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'host', {k: round(v,4) for k,v in h.items()})" >> gpurun_out/${T}_configs.log
  done
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "voxelmap or sync_free or select_variant or small" > gpurun_out/${T}_memcheck.log 2>&1; echo rc=$? >> gpurun_out/${T}_memcheck.log
ls -la gpurun_out | grep ${T}
