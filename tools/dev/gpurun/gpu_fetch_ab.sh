# e2e A/B of the host-filled lower-triangle share (CORR2D_FETCH_FILL_PCT) through
# bench.py's public-call e2e leg, alternating, plus the fetch tests at HEAD.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_fetch.py -q --timeout 300 2>&1 | tail -1
for rep in 1 2; do
  for c in 5 3; do
    for f in 0 25 35; do
      CORR2D_FETCH_FILL_PCT=$f timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/ab/c${c}_f${f}_r$rep.json 2>/dev/null
      python -c "import json;d=json.load(open('gpurun_out/ab/c${c}_f${f}_r$rep.json'));e=d['e2e'];print('cfg$c fill $f rep $rep e2e %.2f ms/call  d2h %.2f GB' % (e['ms_per_step'], e['d2h_bytes_per_step']/1e9))"
    done
  done
done
