# e2e modes: pipelined (default) vs serial, C5 and C3.
set -x
timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_pipe.json 2> gpurun_out/bench_e2e_pipe.err
timeout 500 python bench.py --no-cpu-baseline --e2e-mode pipelined > gpurun_out/bench_e2e_serial.json 2> gpurun_out/bench_e2e_serial.err

