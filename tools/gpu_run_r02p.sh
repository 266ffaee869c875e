# r02p: SM-driven small uploads (no copy-engine queueing), whole-array
# pipelined e2e; GPU tests, bench (serial e2e), bench (pipelined e2e), per-call.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02p_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode pipelined > gpurun_out/r02p_bench_pipe.json 2> gpurun_out/r02p_bench_pipe.err
GVOX_H2D_DMA=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-mode pipelined > gpurun_out/r02p_bench_pipe_dma.json 2> gpurun_out/r02p_bench_pipe_dma.err
GVOX_H2D_DMA=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_bench_dma.json 2> gpurun_out/r02p_bench_dma.err
