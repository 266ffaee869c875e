# r02ae: the register-pipeline linearize variant (probes two points ahead,
# records one point ahead in registers, 3 CTAs/SM) against the base kernel on
# C5 (linearize-only); per-line stall capture of the base kernel.
set -x
T=r02ae
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python tools/variants.py run base,rpipe_b3,rpipe_b2,base,rpipe_b3 > gpurun_out/${T}_variants.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o /tmp/${T}_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_lin.log 2>&1
python tools/ncu_summary.py /tmp/${T}_lin.ncu-rep gpurun_out/${T}_ncu_lin.md > /dev/null 2>&1
ncu -i /tmp/${T}_lin.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_linearize > /tmp/${T}_src.csv 2>/dev/null; gzip -c /tmp/${T}_src.csv > gpurun_out/${T}_src.csv.gz
python tools/ncu_lines.py /tmp/${T}_lin.ncu-rep k_linearize 1.255e10 80 > gpurun_out/${T}_lines.txt 2>&1
GVOX_LIB=paper_2407_10344_b200/build/variants/libgvox_rpipe_b3.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o /tmp/${T}_rp python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_rp.log 2>&1
python tools/ncu_summary.py /tmp/${T}_rp.ncu-rep gpurun_out/${T}_ncu_rp.md > /dev/null 2>&1
ncu -i /tmp/${T}_rp.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_linearize > /tmp/${T}_rsrc.csv 2>/dev/null; gzip -c /tmp/${T}_rsrc.csv > gpurun_out/${T}_rsrc.csv.gz
ls -la gpurun_out | grep ${T}
