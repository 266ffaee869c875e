set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "overlap or select or full_c5 or culling or union or keyframe" > gpurun_out/pytest_ovl.log 2>&1; echo rc=$? >> gpurun_out/pytest_ovl.log
timeout 500 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ovl.json 2> gpurun_out/bench_ovl.err
