# evidence after the planner change: variant-build tests, launch lists and captures -> gpurun_out/
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_checked_build.py tests/test_ct_check.py tests/test_ct_audit.py -m gpu -q 2>&1 | tail -n 4 > gpurun_out/variant_tests.log
timeout 2400 bash tools/reproduce_profiles.sh > gpurun_out/profiles.log 2>&1
python tools/quick_time.py 17669 > gpurun_out/qt17669.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"toom|k1_|k3_|k4_" -s 5 -c 5 -o gpurun_out/mem17669 python tools/quick_time.py 17669 > gpurun_out/ncu_mem17669.log 2>&1
cat gpurun_out/variant_tests.log
