timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_dlr.py tests/test_gpu_lean.py tests/test_gpu_sharded.py tests/test_gpu_dsa_step.py tests/test_gpu_compat.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --more-configs "" --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=sorted(d['ms_per_step_each'])
print('step min/med', e[0], e[len(e)//2], d['ms_per_step'])
"; done
