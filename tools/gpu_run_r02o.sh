# r02o: lifted accumulation (level 0 from the points, coarser levels from the
# finer voxels): GPU tests, build variants, C5 bench, memcheck of the build.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02o_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02o_pytest_gpu.log 2>&1
timeout 900 python tools/variants.py run acc_base,acc_nolift > gpurun_out/r02o_variants_acc.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "voxelmap_parity or sync_free or dense_and_hash" > gpurun_out/r02o_memcheck_build.log 2>&1; echo rc=$? >> gpurun_out/r02o_memcheck_build.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
