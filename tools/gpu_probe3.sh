mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r1c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r1c.log
timeout 300 ./tools/stream_bench > gpurun_out/stream_bench.log 2>&1
( MQ_DBG=$((96 + (100<<8))) KSPLIT=1 timeout 120 python tools/dbg4.py 14336 4096 16;
  MQ_DBG=$((96 + (3<<8))) KSPLIT=1 timeout 120 python tools/dbg4.py 1024 4096 16;
  MQ_DBG=$((96 + (100<<8))) KSPLIT=0 timeout 120 python tools/dbg4.py 14336 4096 16 ) > gpurun_out/dbg4b.log 2>&1
tail -3 gpurun_out/pytest_gpu_r1c.log; cat gpurun_out/stream_bench.log | tail -40
