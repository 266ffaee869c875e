# Screening-kernel variants (stage times from full C5 bench runs).
set -x
timeout 1200 python tools/variants.py run ovl_base,ovl_ilp4_lvs > gpurun_out/variants_ovl.log 2>&1
