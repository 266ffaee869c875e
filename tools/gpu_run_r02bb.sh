# r02bb: candidate order vs locality of the target maps (whole step stages)
set -x
T=r02bb
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for po in source target block8 block32 source block16; do
  GVOX_BENCH_PAIR_ORDER=$po timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$po', round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['stages'].items() if 'ms_per_step' in v and v['ms_per_step']})" >> gpurun_out/${T}_order.log
done
ls -la gpurun_out | grep ${T}
