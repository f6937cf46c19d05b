cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fetch.py -q --timeout 300 > gpurun_out/f_tests.txt 2>&1; echo tests=$?; tail -15 gpurun_out/f_tests.txt
timeout 600 python tools/dev/fetch_probe.py > gpurun_out/f_probe.txt 2>&1; echo probe=$?; cat gpurun_out/f_probe.txt
