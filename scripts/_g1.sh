cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_baseline_parity.py > $O/t7.log 2>&1
timeout 600 python bench.py --steps 8 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 2 > $O/b7.json 2> $O/b7.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l7.csv python scripts/config_steps.py C4 4 > /dev/null 2>&1
