cd $GRAFT_REPO_ROOT
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench2.log 2>&1
