# r02ag: culling loads in one round (27 predicated loads) vs row by row:
# linearize-only and whole-step stage times; parity tests of the culling.
set -x
T=r02ag
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1
timeout 1500 python tools/variants.py run base,cullrows,base,cullrows > gpurun_out/${T}_variants.log 2>&1
timeout 1500 python tools/variants.py run ovl_base,ovl_cullrows,ovl_base,ovl_cullrows > gpurun_out/${T}_variants_ovl.log 2>&1
ls -la gpurun_out | grep ${T}
