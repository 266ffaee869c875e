# Round-2 closing evidence refresh (third session, one B200), after the
# small-call changes that followed r02y: build + smoke, every GPU test with the
# parity-margin records, the C5 bench line, the ncu launch list, the per-config
# table, the NEXT-row benches, the reference arm.  (The kernels of the C5 path
# are those r02y profiled with ncu --set full.)
set -x
T=${TAG:-r02z}
python __graft_entry__.py > gpurun_out/${T}_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
rm -f gpurun_out/${T}_margins.jsonl
GVOX_MARGINS_OUT=gpurun_out/${T}_margins.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 1500 python tools/bench_configs.py ${T} > gpurun_out/${T}_configs_run.log 2>&1
timeout 300 python tools/bench_register.py --reps 20 > gpurun_out/${T}_bench_reg.json 2> gpurun_out/${T}_bench_reg.err
timeout 300 python tools/bench_keyframes.py > gpurun_out/${T}_bench_kf.json 2> gpurun_out/${T}_bench_kf.err
timeout 300 python tools/bench_preprocess.py > gpurun_out/${T}_bench_pre.json 2> gpurun_out/${T}_bench_pre.err
timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global.json 2> gpurun_out/${T}_bench_global.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference_arm.json 2> gpurun_out/${T}_reference_arm.err
ls -la gpurun_out | grep ${T}
