# r02ak: segment-major insert grid (CTAs of many maps resident together)
set -x
T=r02ak
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "voxelmap or sync_free or recycled or lifted or dense" > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python tools/variants.py run acc_base,acc_segmajor0,acc_base,acc_segmajor0 > gpurun_out/${T}_variants.log 2>&1
ls -la gpurun_out | grep ${T}
