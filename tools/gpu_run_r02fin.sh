# r02fin: last check of the committed state -- build + smoke, the GPU suite,
# the default C5 bench line, C2
set -x
T=r02fin
python __graft_entry__.py > gpurun_out/${T}_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 python bench.py --config C2 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
ls -la gpurun_out | grep ${T}
