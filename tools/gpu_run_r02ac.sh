# r02ac: small H2D blocks carried in the launch parameters, host-built tile
# maps for small batches; the whole GPU suite; C1-C3 steps (with / without the
# parameter copies); a per-line stall capture of k_linearize at HEAD.
set -x
T=r02ac
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
for c in C1 C2 C3; do
  for prm in 1 0; do
    GVOX_H2D_PARAM=$prm timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages']; print('$c param=$prm', 'step', round(d['ms_per_step'],4), 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4), 'launches', d['gpu_launches'])" >> gpurun_out/${T}_configs.log
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c2_launches.csv python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_c2_ncu.log 2>&1
timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global.json 2> gpurun_out/${T}_bench_global.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o /tmp/${T}_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_lin.log 2>&1
python tools/ncu_summary.py /tmp/${T}_lin.ncu-rep gpurun_out/${T}_ncu_lin.md > /dev/null 2>&1
ncu -i /tmp/${T}_lin.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_linearize > /tmp/${T}_src.csv 2>/dev/null; gzip -c /tmp/${T}_src.csv > gpurun_out/${T}_src.csv.gz
python tools/ncu_lines.py /tmp/${T}_lin.ncu-rep k_linearize 1.255e10 80 > gpurun_out/${T}_lines.txt 2>&1
ls -la gpurun_out | grep ${T}
