# quick: GPU parity tests + decode timings (development loop)
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
( for k in 0 1; do for s in "14336 4096 16" "4096 4096 16" "1024 4096 16" "6144 4096 16" "4096 14336 16" "28672 4096 16" "28672 8192 16" "4096 4096 1" "14336 4096 64"; do KSPLIT=$k timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done; done ) > gpurun_out/timing_$TAG.log
MQ_DBG=$((96 + (4<<8))) timeout 120 python tools/dbg4.py 4096 4096 16 > gpurun_out/trace_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/timing_$TAG.log
