mkdir -p gpurun_out/d11
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_guards.py -q -x > gpurun_out/d11/guards.log 2>&1
CORR2D_EVIDENCE_DIR=gpurun_out/d11/ev timeout 600 python -m pytest tests/test_gpu_wholemap.py -q > gpurun_out/d11/wholemap.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/d11/gpu_all.log 2>&1
tail -3 gpurun_out/d11/*.log
