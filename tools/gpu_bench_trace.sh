mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1
MQ_DBG=$((96 + (30<<8))) timeout 120 python tools/dbg4.py 14336 4096 16 > gpurun_out/trace_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log | cut -c1-600; head -12 gpurun_out/trace_$TAG.log
