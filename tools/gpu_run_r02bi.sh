# r02bi: C5 e2e with the bulk upload in chunks from a helper thread (the
# library's copies can slip in between), issued at the step start, library
# copies by DMA or SM
set -x
T=r02bi
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
run() {  # label, env...
  lab=$1; shift
  env "$@" timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 15 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lab', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))" >> gpurun_out/${T}_e2e.log
}
run base X=1
run chunk64_early_dma_sm256k GVOX_E2E_CHUNK_MB=64 GVOX_E2E_EARLY_UPLOAD=1 GVOX_H2D_SM_MAX=262144
run chunk64_early_dma GVOX_E2E_CHUNK_MB=64 GVOX_E2E_EARLY_UPLOAD=1 GVOX_H2D_DMA=1
run chunk64_early_sm GVOX_E2E_CHUNK_MB=64 GVOX_E2E_EARLY_UPLOAD=1
run chunk256_early_dma GVOX_E2E_CHUNK_MB=256 GVOX_E2E_EARLY_UPLOAD=1 GVOX_H2D_DMA=1
run chunk64_late_dma GVOX_E2E_CHUNK_MB=64 GVOX_H2D_DMA=1
ls -la gpurun_out | grep ${T}
