# r02aj: overlap culling at the overlap's own level vs the coarsest level;
# parity of the overlap kernels.
set -x
T=r02aj
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
timeout 1500 python tools/variants.py run ovl_base,ovl_cullcoarse,ovl_base,ovl_cullcoarse > gpurun_out/${T}_variants_ovl.log 2>&1
ls -la gpurun_out | grep ${T}
