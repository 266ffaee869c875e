# r02av: C2/C3 e2e with the library's small uploads as kernel parameters or DMA
# (the bulk upload shares PCIe with the SM-driven small copies)
set -x
T=r02av
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for c in C2 C3; do
for mode in base param dma param; do
  unset GVOX_H2D_PARAM GVOX_H2D_DMA
  if [ $mode = param ]; then export GVOX_H2D_PARAM=32000; fi
  if [ $mode = dma ]; then export GVOX_H2D_DMA=1; fi
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --per-call-runs 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $mode', 'step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'per_call', round(d['per_call']['ms_median'],4))" >> gpurun_out/${T}_configs.log
done
done
ls -la gpurun_out | grep ${T}
