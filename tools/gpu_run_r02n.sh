# r02n: kNN lanes-per-query test; compute-sanitizer memcheck / racecheck of the
# r02 memory-management changes (sync-free builds, recycled grids, sentinel
# records, live lists, group kNN).
set -x
timeout 900 python -m pytest tests/test_gpu_preprocess.py -q -x > gpurun_out/r02n_pytest_pre.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "sync_free or recycled or c2_validation or c1 or select_equals_two_calls and 1-20" > gpurun_out/r02n_memcheck_parity.log 2>&1; echo rc=$? >> gpurun_out/r02n_memcheck_parity.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_preprocess.py -q -x -k "lanes_per_query and 10" > gpurun_out/r02n_memcheck_knn.log 2>&1; echo rc=$? >> gpurun_out/r02n_memcheck_knn.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_validation or c1" > gpurun_out/r02n_racecheck_linearize.log 2>&1; echo rc=$? >> gpurun_out/r02n_racecheck_linearize.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_global.py tests/test_gpu_keyframes.py -q -x > gpurun_out/r02n_memcheck_next.log 2>&1; echo rc=$? >> gpurun_out/r02n_memcheck_next.log
