for v in 1 0 1 0; do
  DLRSN_STEP_FORK=$v python bench.py --full-sn 0 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('fork=$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
