# Linearize-kernel variants (C5, bench.py --linearize-only).
set -x
timeout 1200 python tools/variants.py run base,branchless > gpurun_out/variants_lin.log 2>&1
