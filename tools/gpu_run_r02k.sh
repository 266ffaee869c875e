# r02k: cluster PCG (tests + NEXT-4 bench + ncu), C2 build host laps.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02k_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02k_pytest_gpu.log 2>&1
timeout 600 python tools/bench_global.py > gpurun_out/r02k_bench_global.json 2> gpurun_out/r02k_bench_global.err
GVOX_PCG_CLUSTER_MB=0 timeout 600 python tools/bench_global.py > gpurun_out/r02k_bench_global_grid.json 2> gpurun_out/r02k_bench_global_grid.err
GVOX_DEBUG_TIMING=1 timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > /dev/null 2> gpurun_out/r02k_c2_build_laps.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg -c 1 -o gpurun_out/r02k_pcg python tools/bench_global.py > gpurun_out/r02k_ncu_pcg.log 2>&1
