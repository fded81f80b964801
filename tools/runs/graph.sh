cd "$GRAFT_REPO_ROOT"; python tools/graph_step.py 17669 > gpurun_out/graph.log 2>&1; python tools/graph_step.py 35851 >> gpurun_out/graph.log 2>&1
