# r02v: grid-strided cloud packing (tests, pack time, e2e)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02v_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02v_pytest_gpu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02v_pack_launches.csv -k regex:k_cloud_pack python bench.py --steps 1 --warmup 3 --no-cpu-baseline --per-call-runs 0 --e2e-steps 2 > gpurun_out/r02v_ncu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err
