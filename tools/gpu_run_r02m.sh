# r02m: group kNN with G CTAs per tile (G x more threads per frame).
set -x
timeout 900 python -m pytest tests/test_gpu_preprocess.py -q -x > gpurun_out/r02m_pytest_pre.log 2>&1
for g in 1 4 8; do GVOX_KNN_GROUP=$g timeout 300 python tools/bench_preprocess.py > gpurun_out/r02m_pre_g$g.json 2> gpurun_out/r02m_pre_g$g.err; done
for g in 4 8; do GVOX_KNN_GROUP=$g timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_knn_query -c 1 -o gpurun_out/r02m_knn_g$g python tools/bench_preprocess.py > gpurun_out/r02m_ncu_knn_g$g.log 2>&1; done
