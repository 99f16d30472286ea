cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2; do for c in head nodiag diag; do DLRSN_LIB=scratch/lib_$c.so timeout 600 python bench.py --steps 6 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step_each'][2:], d['roofline']['launch_ms'])"; done; done > $O/ab_k3.log 2>&1
