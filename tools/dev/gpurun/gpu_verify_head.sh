cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/v_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/v_gputests.txt 2>&1; echo tests=$?; tail -3 gpurun_out/v_gputests.txt
for c in 5 1 2 3; do timeout 900 python bench.py --config $c > gpurun_out/v_bench_cfg$c.json 2> gpurun_out/v_bench_cfg$c.err; echo cfg$c=$?; tail -1 gpurun_out/v_bench_cfg$c.json | cut -c1-300; done
timeout 900 python bench.py --impl reference > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; echo ref=$?; tail -1 gpurun_out/v_ref.json | cut -c1-300
