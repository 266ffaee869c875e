# Screening-kernel variants (stage times from full C5 bench runs).
set -x
timeout 1200 python tools/variants.py run acc_base,acc_acc4_ins6,acc_acc4_ins8,acc_acc4_ins6_fin > gpurun_out/variants_ovl.log 2>&1
