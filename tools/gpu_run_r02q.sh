# r02q: default bench (pipelined e2e over 10 steps, pinned result buffer) and
# the serial e2e for comparison.
set -x
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode serial --e2e-steps 5 > gpurun_out/r02q_bench_serial.json 2> gpurun_out/r02q_bench_serial.err
GVOX_E2E_DEBUG=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 4 > /dev/null 2> gpurun_out/r02q_e2e_debug.log
