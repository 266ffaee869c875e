# Screening-kernel variants (stage times from full C5 bench runs).
set -x
timeout 1200 python tools/variants.py run acc_base,acc_seg2,acc_seg3 > gpurun_out/variants_ovl.log 2>&1
