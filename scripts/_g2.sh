cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 3600 python scripts/parity_long.py C3 100 $O/r02_parity_long_c3.json > $O/plong_c3.log 2>&1
timeout 1500 python scripts/parity_long.py C4 12 $O/r02_parity_long_c4.json > $O/plong_c4.log 2>&1
