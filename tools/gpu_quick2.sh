mkdir -p gpurun_out
TAG=${1:-q}
( for s in "14336 4096 16" "4096 4096 16" "1024 4096 16" "6144 4096 16" "4096 14336 16" "28672 4096 16" "28672 8192 16"; do timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done ) > gpurun_out/timing_$TAG.log
MQ_DBG=$((96 + (4<<8))) timeout 120 python tools/dbg4.py 4096 4096 16 > gpurun_out/trace_$TAG.log 2>&1
cat gpurun_out/timing_$TAG.log gpurun_out/trace_$TAG.log
