cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python bench.py --steps 8 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 2 > $O/b6.json 2> $O/b6.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l6.csv python scripts/config_steps.py C4 4 > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/t6.log 2>&1
