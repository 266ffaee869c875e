# ncu --set full of the build and screening kernels at full C5 (one launch each).
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_build_accum|k_build_insert|k_overlap_select|k_build_finalize" -c 4 -o gpurun_out/prof_build_c5_g python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_build.log 2>&1
