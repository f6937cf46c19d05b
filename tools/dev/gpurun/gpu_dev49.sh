cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_bench_multirank.py -x -q --timeout 150 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_bench_multirank.py -x -q --timeout 150 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
