# r02y: L1 prefetch of the next point's records: tests, variants, ncu
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02y_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02y_pytest_gpu.log 2>&1
timeout 900 python tools/variants.py run base,lin_noprefetch > gpurun_out/r02y_variants_lin.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o gpurun_out/r02y_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/r02y_ncu_lin.log 2>&1
