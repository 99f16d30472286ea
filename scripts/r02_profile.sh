#!/bin/bash
# Round-2 C4 captures: launch list of 4 steps, then one --set full capture
# of K3 and of the DLR sweep (each after the plain run exited 0).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python scripts/config_steps.py C4 4 > $O/c4_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/r02_c4_launches.csv python scripts/config_steps.py C4 4 > $O/c4_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_mma32 \
  --launch-skip 2 -c 1 -o $O/r02_c4_k3 python scripts/config_steps.py C4 4 > $O/c4_ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel \
  --launch-skip 8 -c 1 -o $O/r02_c4_sweep python scripts/config_steps.py C4 4 > $O/c4_ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:phi_quadrant \
  --launch-skip 8 -c 1 -o $O/r02_c4_phiq python scripts/config_steps.py C4 4 > $O/c4_ncu_phiq.log 2>&1
ls -la $O
