# Round-end style check: build, smoke, all GPU tests, the C5 bench line, ncu
# launch list, one ncu --set full capture of k_linearize at full C5.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_linearize" -c 1 -o gpurun_out/prof_lin_c5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lin.log 2>&1
