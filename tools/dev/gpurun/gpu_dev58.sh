cd $GRAFT_REPO_ROOT
export BENCH_ONE_DEVICE=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/mr5.out 2> gpurun_out/mr5.err
echo rc $?
tail -1 gpurun_out/mr5.out | cut -c1-600; grep -v "^W10" gpurun_out/mr5.err | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 --steps 5 --warmup 3 --impl reference > gpurun_out/mr5r.out 2> gpurun_out/mr5r.err
echo rc $?
tail -1 gpurun_out/mr5r.out | cut -c1-300
