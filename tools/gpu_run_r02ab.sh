# r02ab: kNN (top-k list in registers, fp32 pre-filter, k <= 10 lists) and
# the two-barrier persistent PCG: parity tests, timings against the previous
# kernels (env knobs), ncu of each; the C2 step's launch list.
set -x
T=r02ab
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_preprocess.py tests/test_gpu_global.py -q -x > gpurun_out/${T}_pytest_next.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "select" > gpurun_out/${T}_pytest_select.log 2>&1
for g in 1 4 8; do GVOX_KNN_GROUP=$g timeout 300 python tools/bench_preprocess.py > gpurun_out/${T}_pre_g$g.json 2> gpurun_out/${T}_pre_g$g.err; done
timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global.json 2> gpurun_out/${T}_bench_global.err
GVOX_PCG_BARRIERS=4 timeout 600 python tools/bench_global.py > gpurun_out/${T}_bench_global_4bar.json 2> gpurun_out/${T}_bench_global_4bar.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_knn_query -c 1 -o /tmp/${T}_knn python tools/bench_preprocess.py > gpurun_out/${T}_ncu_knn.log 2>&1
python tools/ncu_summary.py /tmp/${T}_knn.ncu-rep gpurun_out/${T}_ncu_knn.md > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg -c 1 -o /tmp/${T}_pcg python tools/bench_global.py > gpurun_out/${T}_ncu_pcg.log 2>&1
python tools/ncu_summary.py /tmp/${T}_pcg.ncu-rep gpurun_out/${T}_ncu_pcg.md > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c2_launches.csv python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_c2_ncu.log 2>&1
timeout 300 python bench.py --config C2 --steps 50 --no-cpu-baseline --per-call-runs 20 > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
GVOX_DEBUG_TIMING=1 timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/${T}_c2_dbg.json 2> gpurun_out/${T}_c2_dbg.err
ls -la gpurun_out | grep ${T}
