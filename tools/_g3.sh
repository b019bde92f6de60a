cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q --timeout 300 > gpurun_out/gputest_sk.log 2>&1; echo rc=$? >> gpurun_out/gputest_sk.log
timeout 200 python tools/graph_time.py 16 > gpurun_out/graph_sk.txt 2>&1
timeout 200 python tools/graph_time.py 1 >> gpurun_out/graph_sk.txt 2>&1
SCHED=1 timeout 200 python tools/graph_time.py 16 >> gpurun_out/graph_sk.txt 2>&1
SCHED=2 timeout 200 python tools/graph_time.py 16 >> gpurun_out/graph_sk.txt 2>&1
timeout 100 python tools/stack_time.py 1 16 32 >> gpurun_out/graph_sk.txt 2>&1
