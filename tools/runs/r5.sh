cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_ct_check.py tests/test_checked_build.py -q -m gpu -rfEs > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
timeout 600 python tools/kernel_times.py 57637:16384 35851 > gpurun_out/kt5.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2201_10473_b200.ct_check import ct_check
import json
for b in (32, 4096):
    print(json.dumps(ct_check(batch=b, trials=2000)))
" > gpurun_out/ct5.log 2>&1
F2X_LIB_VARIANT=leaky python -c "
import sys; sys.path.insert(0,'.')
from paper_2201_10473_b200.ct_check import ct_check
import json
for b in (32, 4096):
    print(json.dumps(ct_check(batch=b, trials=2000)))
" >> gpurun_out/ct5.log 2>&1
