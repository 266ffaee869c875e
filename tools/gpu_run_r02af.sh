# r02af: level-major build slots, fused PCG dot products, the FAST pipeline's
# order inside a live iteration (variants), PCG grid sizes; whole GPU suite.
set -x
T=r02af
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
timeout 1500 python tools/variants.py run base,order1,order2,base,order1 > gpurun_out/${T}_variants.log 2>&1
timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global.json 2> gpurun_out/${T}_bench_global.err
for c in 32 64; do GVOX_PCG_CTAS=$c timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global_ctas$c.json 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
ls -la gpurun_out | grep ${T}
