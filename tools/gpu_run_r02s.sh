# r02s: e2e with device-kept screening decisions vs host decisions; debug laps.
set -x
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --per-call-runs 0 > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
GVOX_E2E_HOST_SELECT=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --per-call-runs 0 > gpurun_out/r02s_bench_hostsel.json 2> gpurun_out/r02s_bench_hostsel.err
GVOX_E2E_DEBUG=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 4 > /dev/null 2> gpurun_out/r02s_e2e_debug.log
