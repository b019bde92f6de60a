cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_weight_quant.py -x -q --timeout 300 > gpurun_out/gputest_wq.log 2>&1; echo rc=$? >> gpurun_out/gputest_wq.log
