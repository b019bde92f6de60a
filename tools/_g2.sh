cd $GRAFT_REPO_ROOT
timeout 60 ./tools/microbench/stream_graph > gpurun_out/stream_graph.txt 2>&1
timeout 200 python tools/graph_time.py 16 > gpurun_out/graph_time16.txt 2>&1
for pf in "" 0 8 32; do if [ -z "$pf" ]; then timeout 200 python tools/stack_time.py 1 16 64; else PF=$pf timeout 200 python tools/stack_time.py 1 16 64; fi; done > gpurun_out/stack_pf.txt 2>&1
