cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2; do for f in 0 1; do DLRSN_STEP_FORK=$f timeout 900 python bench.py --steps 20 --warmup 5 --more-configs "C2,C3" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fork $f', round(d['ms_per_step'],3), max(d['ms_per_step_each']), [round(m['ms_per_step'],3) for m in d['more_configs']], d['clocks']['samples'])"; done; done > $O/fork2.log 2>&1
