# r02c: new bench line, ncu of k_linearize (full set, source), launch list,
# shard model, 2-rank gloo plumbing bench, dist GPU tests.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/r02c_pytest_dist.log 2>&1
GVOX_DIST_BACKEND=gloo GVOX_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --submaps 100 --no-e2e > gpurun_out/r02c_bench_2rank_gloo.json 2> gpurun_out/r02c_bench_2rank_gloo.err
timeout 900 ncu --set full --import-source on -k regex:k_linearize -c 1 --launch-skip 3 -o gpurun_out/r02c_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/r02c_ncu_lin.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-call-runs 0 > gpurun_out/r02c_ncu_bench.log 2>&1
timeout 1200 python tools/shard_model.py > gpurun_out/r02c_shard_model.json 2> gpurun_out/r02c_shard_model.err
ls -la gpurun_out
