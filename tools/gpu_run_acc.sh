# Build-accumulation variants (stage times from full C5 bench runs) + voxel-map parity.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "voxelmap or dense or golden" > gpurun_out/pytest_acc.log 2>&1; echo rc=$? >> gpurun_out/pytest_acc.log
timeout 1200 python tools/variants.py run acc_base,acc_r01f,acc_nohoist,acc_nomaxrun,acc_seg2,acc_seg3 > gpurun_out/variants_acc.log 2>&1
