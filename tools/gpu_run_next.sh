python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_global.py tests/test_gpu_preprocess.py -q > gpurun_out/pytest_g2.log 2>&1; echo rc=$? >> gpurun_out/pytest_g2.log
timeout 300 python tools/bench_preprocess.py > gpurun_out/bench_pre.json 2> gpurun_out/bench_pre.err
timeout 300 python tools/bench_global.py > gpurun_out/bench_global.json 2> gpurun_out/bench_global.err
GVOX_PCG_GRAPH=1 timeout 300 python tools/bench_global.py > gpurun_out/bench_global_graph.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linearize -c 1 -o gpurun_out/prof_r01e_lin python bench.py --linearize-only --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/pytest_g2.log; cat gpurun_out/bench_pre.json gpurun_out/bench_global.json gpurun_out/bench_global_graph.json; tail -n 2 gpurun_out/ncu_full.log
