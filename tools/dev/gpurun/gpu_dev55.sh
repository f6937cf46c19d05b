cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
for c in 1 2; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none -k regex:"small_" -s 400 -c 4 --csv python tools/dev/small_rot.py $c 16 > gpurun_out/prof2/traffic_cfg$c.csv 2>gpurun_out/prof2/traffic_cfg$c.err
done
grep -v "^==" gpurun_out/prof2/traffic_cfg1.csv | cut -c1-250 | tail -14
