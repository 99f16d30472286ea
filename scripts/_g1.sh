cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2 3 4; do DLRSN_GRAPH_DEBUG=1 timeout 600 python bench.py --steps 20 --warmup 5 --more-configs "" --no-cpu-baseline --e2e-steps 1 2> $O/clk_err_$rep.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step_each'], d['si_iterations'])"; grep -c capture $O/clk_err_$rep.log; done > $O/clk2.log 2>&1
