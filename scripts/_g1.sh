cd $GRAFT_REPO_ROOT
O=gpurun_out
for ns in 0 1 2 3; do DLRSN_K3_WS=0 DLRSN_K3_NOSTAGE=$ns timeout 600 python bench.py --steps 3 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nostage $ns', d['roofline']['launch_ms'])"; done > $O/nostage2.log 2>&1
