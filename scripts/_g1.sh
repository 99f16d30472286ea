cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_baseline_parity.py > $O/t12.log 2>&1
timeout 600 python bench.py --steps 8 --warmup 3 --more-configs "" --no-cpu-baseline --e2e-steps 2 > $O/b12.json 2> $O/b12.err
