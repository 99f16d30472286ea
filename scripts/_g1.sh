cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dlr.py tests/test_gpu_slab.py -x -q > $O/t17.log 2>&1
for rep in 1 2; do for c in nodiag half; do DLRSN_LIB=scratch/lib_$c.so timeout 600 python bench.py --steps 6 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step_each'][2:], d['roofline']['launch_ms'])"; done; done > $O/ab_k3b.log 2>&1
