#!/bin/bash
# ncu --set full captures of the new CholQR2 kernels (after the plain run exited 0)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python scripts/config_steps.py C4 4 > $O/c4_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mgram64s \
  --launch-skip 2 -c 1 -f -o $O/r02c_c4_mgram64s python scripts/config_steps.py C4 4 > $O/c4_ncu_mg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowmix_upper_pipe \
  --launch-skip 2 -c 1 -f -o $O/r02c_c4_rowmix_upper_pipe python scripts/config_steps.py C4 4 > $O/c4_ncu_ru.log 2>&1
ls -la $O/*.ncu-rep
