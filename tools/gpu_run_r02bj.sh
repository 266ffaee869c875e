# r02bj: k-NN with 16 lanes per query (one frame) vs 8; preprocessing tests
set -x
T=r02bj
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_preprocess.py -q -x > gpurun_out/${T}_pytest.log 2>&1
for g in 8 16 8 16; do GVOX_KNN_GROUP=$g timeout 300 python tools/bench_preprocess.py 2>/dev/null | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('G=$g', d['workload'], round(d['knn_device_ms'],4))" >> gpurun_out/${T}_knn.log; done
ls -la gpurun_out | grep ${T}
