# Round-end style run: build, smoke, all GPU tests, the C5 bench line, per-config
# table, ncu launch list, memcheck of the screened-batch path.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x -k "linearize_select_equals and 1-20" > gpurun_out/memcheck_select.log 2>&1; echo rc=$? >> gpurun_out/memcheck_select.log
ls -la gpurun_out
