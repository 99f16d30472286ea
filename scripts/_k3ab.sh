for cfg in "1 296" "1 592" "1 1184" "0 1776" "0 3552"; do set -- $cfg; echo "== SEQ=$1 RANGES=$2"; DLRSN_K3_SEQ=$1 DLRSN_K3_RANGES=$2 timeout 300 python bench.py --steps 8 --warmup 4 --more-configs "" --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=sorted(d['ms_per_step_each'])
print('step min/med', e[0], e[len(e)//2], 'K3', d['roofline']['launch_ms'], d['si_iterations'])
"; done
echo "== old"; DLRSN_K3_D64=0 timeout 300 python bench.py --steps 8 --warmup 4 --more-configs "" --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=sorted(d['ms_per_step_each'])
print('step min/med', e[0], e[len(e)//2], 'K3', d['roofline']['launch_ms'], d['si_iterations'])
"
