#!/bin/bash
# Round-2 (second half) C4 captures with the diagonal-block K3: launch list of
# 4 steps, then one --set full capture of K3 (each after the plain run exited 0).
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python scripts/config_steps.py C4 4 > $O/c4_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/r02b_c4_launches.csv python scripts/config_steps.py C4 4 > $O/c4_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_mma64d \
  --launch-skip 2 -c 1 -f -o $O/r02b_c4_k3d64 python scripts/config_steps.py C4 4 > $O/c4_ncu_k3.log 2>&1
ls -la $O
