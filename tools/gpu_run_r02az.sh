# r02az: tiles of up to 32k points for every factor (at least 1 tile) vs 2
set -x
T=r02az
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python tools/variants.py run base,tmin1,base,tmin1 > gpurun_out/${T}_variants.log 2>&1
ls -la gpurun_out | grep ${T}
