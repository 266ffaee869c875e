# Build-kernel change check: voxel-map parity tests, the C5 bench line, and one
# ncu --set full capture of the build and screening kernels at full C5.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "voxelmap or full_c5 or select or dense" > gpurun_out/pytest_build.log 2>&1; echo rc=$? >> gpurun_out/pytest_build.log
timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_build_accum|k_build_insert|k_overlap_select|k_build_finalize" -c 4 -o gpurun_out/prof_build_c5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_build.log 2>&1
