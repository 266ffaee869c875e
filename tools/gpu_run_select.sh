# Fused screening -> linearization check: the new parity tests, then the C5 bench line.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "select or full_c5" > gpurun_out/pytest_select.log 2>&1; echo rc=$? >> gpurun_out/pytest_select.log
timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench_sel.json 2> gpurun_out/bench_sel.err
