# r02u: ncu --set full of the cloud packing kernel (e2e clouds phase)
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cloud_pack -c 1 -o gpurun_out/r02u_pack python bench.py --steps 1 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 1 > gpurun_out/r02u_ncu.log 2>&1
