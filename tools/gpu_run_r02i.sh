# r02i: fused-Omega level term (default) + dyadic-templated screening: GPU
# tests, linearize variants (warp-level level skip, early gathers), bench line.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02i_pytest_gpu.log 2>&1
timeout 1200 python tools/variants.py run base,lin_nofuse,lin_wskip,lin_early,lin_early_wskip > gpurun_out/r02i_variants_lin.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
