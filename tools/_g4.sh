cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 200 python tools/graph_time.py 16 > gpurun_out/graph_time16.txt 2>&1
timeout 200 python tools/graph_time.py 1 >> gpurun_out/graph_time16.txt 2>&1
timeout 200 python tools/stack_time.py 1 16 32 64 > gpurun_out/stack.txt 2>&1
