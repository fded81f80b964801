cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" leaky; do
F2X_LIB_VARIANT=$v python -c "
import sys; sys.path.insert(0,'.')
from paper_2201_10473_b200.ct_check import ct_check
import json
print(json.dumps(ct_check(trials=4000)))
print(json.dumps(ct_check(trials=4000, control=True)))
print(json.dumps(ct_check(trials=4000, seed=0xC9)))
"
done > gpurun_out/ct6.log 2>&1
