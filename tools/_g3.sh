cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q --timeout 400 > gpurun_out/gputest_sh.log 2>&1; echo rc=$? >> gpurun_out/gputest_sh.log
