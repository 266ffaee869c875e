# r02f: nested dense grids + cheaper pipeline bookkeeping (+ barrier-free
# screening): GPU tests, linearize variants, bench line.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02f_pytest_gpu.log 2>&1
timeout 900 python tools/variants.py run base,lin_nonest,lin_incbase > gpurun_out/r02f_variants_lin.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
