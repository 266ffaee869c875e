# r02t: where the e2e clouds phase goes (build laps), pack kernel time (ncu launch list)
set -x
GVOX_DEBUG_TIMING=1 GVOX_E2E_DEBUG=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 3 > /dev/null 2> gpurun_out/r02t_e2e_debug.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_e2e_launches.csv -k regex:k_cloud_pack python bench.py --steps 1 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 2 > gpurun_out/r02t_ncu.log 2>&1
