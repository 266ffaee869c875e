# r02e: barrier-free screening kernel (tests + variants), fresh ncu captures
# (clock-control none) of k_linearize and of the build / screening kernels.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02e_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_pytest_gpu.log 2>&1
timeout 900 python tools/variants.py run ovl_bar,ovl_nobar,ovl_nobar_b6,ovl_nobar_b8 > gpurun_out/r02e_variants_ovl.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o gpurun_out/r02e_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/r02e_ncu_lin.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_build|k_overlap_select" -c 4 --launch-skip 8 -o gpurun_out/r02e_bo python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/r02e_ncu_bo.log 2>&1
