# Round-2 final evidence run (third session, one B200): build + smoke, every
# GPU test with the parity-margin records, the C5 bench line, the ncu launch
# list of the bench command, ncu --set full of the dominant kernel (with the
# per-line stall summary) and of the build / screening kernels, the per-config
# table, 2-rank gloo plumbing runs of bench.py, the NEXT-row benches and the
# reference arm.  Everything lands in gpurun_out/${TAG}_*.
set -x
T=${TAG:-r02y}
python __graft_entry__.py > gpurun_out/${T}_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
rm -f gpurun_out/${T}_margins.jsonl
GVOX_MARGINS_OUT=gpurun_out/${T}_margins.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o gpurun_out/${T}_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_lin.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_lin.ncu-rep gpurun_out/${T}_ncu_linearize_c5.md > /dev/null 2>&1
ncu -i gpurun_out/${T}_lin.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_linearize 2>/dev/null | gzip -c > /tmp/${T}_src.csv.gz; python tools/ncu_stalls.py /tmp/${T}_src.csv.gz 30 > gpurun_out/${T}_stalls_linearize.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_build|k_overlap_select" -c 5 --launch-skip 10 -o gpurun_out/${T}_bo python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_bo.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_bo.ncu-rep gpurun_out/${T}_ncu_build_overlap_c5.md > /dev/null 2>&1
timeout 1500 python tools/bench_configs.py ${T} > gpurun_out/${T}_configs_run.log 2>&1
GVOX_DIST_BACKEND=gloo GVOX_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 3 --warmup 3 --submaps 100 --no-e2e > gpurun_out/${T}_bench_2rank_gloo_c5.json 2> gpurun_out/${T}_bench_2rank_gloo_c5.err
GVOX_DIST_BACKEND=gloo GVOX_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 5 --warmup 3 --config C2 > gpurun_out/${T}_bench_2rank_gloo_c2.json 2> gpurun_out/${T}_bench_2rank_gloo_c2.err
timeout 300 python tools/bench_register.py --reps 20 > gpurun_out/${T}_bench_reg.json 2> gpurun_out/${T}_bench_reg.err
timeout 300 python tools/bench_keyframes.py > gpurun_out/${T}_bench_kf.json 2> gpurun_out/${T}_bench_kf.err
timeout 300 python tools/bench_preprocess.py > gpurun_out/${T}_bench_pre.json 2> gpurun_out/${T}_bench_pre.err
timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global.json 2> gpurun_out/${T}_bench_global.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference_arm.json 2> gpurun_out/${T}_reference_arm.err
ls -la gpurun_out | grep ${T}
