cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/final_b200.json 2> gpurun_out/final_b200.err; tail -1 gpurun_out/final_b200.json | cut -c1-400
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -1 gpurun_out/final_ref.json | cut -c1-300
