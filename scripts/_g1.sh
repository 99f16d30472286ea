cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/step_probe.py C3 14 > $O/probe4.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_baseline_parity.py > $O/t10.log 2>&1
timeout 600 python bench.py --steps 8 --warmup 3 --more-configs "C2,C3" --no-cpu-baseline --e2e-steps 2 > $O/b10.json 2> $O/b10.err
