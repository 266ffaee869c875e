# r02r: PCG with row chunks (tests, C4 timing vs one chunk per row, ncu),
# e2e without the unused normals for C5.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02r_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02r_pytest_gpu.log 2>&1
timeout 600 python tools/bench_global.py > gpurun_out/r02r_bench_global.json 2> gpurun_out/r02r_bench_global.err
GVOX_PCG_CHUNK=0 timeout 600 python tools/bench_global.py > gpurun_out/r02r_bench_global_rows.json 2> gpurun_out/r02r_bench_global_rows.err
GVOX_PCG_CHUNK=32 timeout 600 python tools/bench_global.py > gpurun_out/r02r_bench_global_c32.json 2> gpurun_out/r02r_bench_global_c32.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg -c 1 -o gpurun_out/r02r_pcg python tools/bench_global.py > gpurun_out/r02r_ncu_pcg.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
