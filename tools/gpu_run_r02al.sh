# r02al: the insert records the voxel indices it already knows (the
# accumulation skips their grid reads)
set -x
T=r02al
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
timeout 1500 python tools/variants.py run acc_base,acc_known0,acc_base,acc_known0 > gpurun_out/${T}_variants.log 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:k_build_insert|k_build_accum" -c 2 --launch-skip 6 -o /tmp/${T}_b python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_b.log 2>&1
python tools/ncu_summary.py /tmp/${T}_b.ncu-rep gpurun_out/${T}_ncu_build.md > /dev/null 2>&1
ls -la gpurun_out | grep ${T}
