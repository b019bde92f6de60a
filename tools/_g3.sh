cd $GRAFT_REPO_ROOT
timeout 200 python tools/graph_time.py 16 > gpurun_out/early.txt 2>&1
timeout 100 python tools/stack_time.py 1 16 64 256 512 >> gpurun_out/early.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/gputest_all.log 2>&1; echo rc=$? >> gpurun_out/gputest_all.log
