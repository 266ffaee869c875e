# r02aa: screened-batch variant from the selected candidates (tests), hit
# statistics of the C5 workload, and a per-source-line ncu capture of
# k_linearize at HEAD (the baseline for this session's kernel work).
set -x
T=r02aa
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "select" > gpurun_out/${T}_pytest_select.log 2>&1
timeout 600 python tools/hitfrac.py > gpurun_out/${T}_hitfrac.log 2>&1
timeout 300 python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_lin.json 2> gpurun_out/${T}_lin.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_linearize -c 1 --launch-skip 3 -o /tmp/${T}_lin python bench.py --linearize-only --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --per-call-runs 0 > gpurun_out/${T}_ncu_lin.log 2>&1
python tools/ncu_lines.py /tmp/${T}_lin.ncu-rep k_linearize 1.255e10 80 > gpurun_out/${T}_lines.txt 2>&1
python tools/sass_hist.py /tmp/${T}_lin.ncu-rep k_linearize 1.255e10 > gpurun_out/${T}_sass_hist.txt 2>&1
python tools/ncu_summary.py /tmp/${T}_lin.ncu-rep gpurun_out/${T}_ncu_lin.md > gpurun_out/${T}_ncu_sum.log 2>&1
ncu -i /tmp/${T}_lin.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_linearize > /tmp/${T}_src.csv 2>/dev/null; gzip -c /tmp/${T}_src.csv > gpurun_out/${T}_src.csv.gz
ncu -i /tmp/${T}_lin.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>&1
ls -la gpurun_out | grep ${T}
