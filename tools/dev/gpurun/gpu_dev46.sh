cd $GRAFT_REPO_ROOT
export BENCH_ONE_DEVICE=1
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --config 2 --steps 2 --warmup 3 --spectra broadcast > gpurun_out/mr.out 2> gpurun_out/mr.err
echo rc $?
tail -5 gpurun_out/mr.out; tail -30 gpurun_out/mr.err
