cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dlr.py -x -q -k "twenty" > $O/t21.log 2>&1
