cd $GRAFT_REPO_ROOT
export BENCH_ONE_DEVICE=1 PYTHONFAULTHANDLER=1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --config 2 --steps 2 --warmup 3 --spectra broadcast > gpurun_out/mr.out 2> gpurun_out/mr.err &
TR=$!
for i in $(seq 1 90); do sleep 1; if ! kill -0 $TR 2>/dev/null; then echo "finished after $i s"; break; fi; done
if kill -0 $TR 2>/dev/null; then
  for c in $(pgrep -P $TR); do kill -ABRT $c; done
  sleep 5; kill $TR 2>/dev/null
fi
wait $TR; echo rc $?
grep -v "^W1020\|^ *$" gpurun_out/mr.err | grep -B2 -A30 "Thread\|Current thread" | head -120
tail -3 gpurun_out/mr.out
