# r02ah: culling pass with the next pass's chunk boxes prefetched
set -x
T=r02ah
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${T}_pytest_parity.log 2>&1
timeout 1500 python tools/variants.py run base,cullpf0,cull27pf,base,cullpf0 > gpurun_out/${T}_variants.log 2>&1
ls -la gpurun_out | grep ${T}
