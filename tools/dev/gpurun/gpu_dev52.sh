cd $GRAFT_REPO_ROOT
(nvidia-smi -i 0 --query-gpu=index,clocks.sm --format=csv,noheader,nounits -lms 100 > /dev/null 2>&1 &) 
sleep 1
timeout 120 python tools/dev/small_rot.py 1 200 32 2>&1 | tail -3
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_1808_00685_b200 as P
from paper_1808_00685_b200 import api, configs as C
case = C.make(1)
import bench
spec = bench.__dict__.get('make_spec')
print([k for k in dir(case) if not k.startswith('_')])
print(case.resample, case.alpha, case.interpolant)
PY
