cd $GRAFT_REPO_ROOT
export BENCH_ONE_DEVICE=1 PYTHONFAULTHANDLER=1
for it in 1 2 3 4 5 6; do
port=$((29600 + it))
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --config 2 --steps 2 --warmup 3 --spectra broadcast > gpurun_out/mr$it.out 2> gpurun_out/mr$it.err &
TR=$!
done_=0
for i in $(seq 1 60); do sleep 1; if ! kill -0 $TR 2>/dev/null; then echo "it $it finished after $i s"; done_=1; break; fi; done
if [ $done_ = 0 ]; then
  echo "it $it HUNG"; for c in $(pgrep -P $TR); do kill -ABRT $c; done
  sleep 5; kill $TR 2>/dev/null; wait $TR
  grep -v "^W1020" gpurun_out/mr$it.err | grep -A25 "most recent call first" | head -80
  break
fi
wait $TR
done
