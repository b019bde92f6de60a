mkdir -p gpurun_out
TAG=${1:-p}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python tools/quick_time.py prefill > gpurun_out/quickpf_$TAG.log 2>&1
timeout 300 python tools/quick_time.py > gpurun_out/quick_$TAG.log 2>&1
tail -2 gpurun_out/pytest_$TAG.log; cat gpurun_out/quickpf_$TAG.log gpurun_out/quick_$TAG.log
