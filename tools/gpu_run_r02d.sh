# r02d: FAST-pipeline bookkeeping rewrite (live-iteration list, strided copy
# addresses, sentinel records): GPU tests, linearize-only timing, bench line.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02d_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02d_pytest_gpu.log 2>&1
timeout 600 python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 6 --per-call-runs 0 > gpurun_out/r02d_linonly.json 2> gpurun_out/r02d_linonly.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
