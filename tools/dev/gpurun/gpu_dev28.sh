cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:small_stream -s 5 -c 1 -o gpurun_out/stream2 python tools/one_small.py 2 > gpurun_out/ncu28.log 2>&1
tail -3 gpurun_out/ncu28.log
