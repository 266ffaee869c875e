# r02aq: k-NN lanes per query on one frame (G = 4 / 8 / 16) and PCG row-chunk
# sizes with the two-barrier kernel
set -x
T=r02aq
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for g in 4 8 4 8; do GVOX_KNN_GROUP=$g timeout 300 python tools/bench_preprocess.py 2>/dev/null | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('G=$g', d['workload'], round(d['knn_device_ms'],4))" >> gpurun_out/${T}_knn.log; done
for c in 32 64 128 64; do GVOX_PCG_CHUNK=$c timeout 600 python tools/bench_global.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk=$c', round(d['solve_ms'],3), d['pcg_iterations'])" >> gpurun_out/${T}_pcg.log; done
ls -la gpurun_out | grep ${T}
