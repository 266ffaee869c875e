# Linearize-kernel variants (C5, bench.py --linearize-only).
set -x
timeout 1200 python tools/variants.py run base,t96_b5,t96_b6,t160_b3 > gpurun_out/variants_lin.log 2>&1
