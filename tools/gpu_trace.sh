mkdir -p gpurun_out
( MQ_DBG=$((96 + (100<<8))) KSPLIT=1 timeout 120 python tools/dbg4.py 14336 4096 16;
  MQ_DBG=$((96 + (5<<8))) KSPLIT=1 timeout 120 python tools/dbg4.py 14336 4096 16;
  MQ_DBG=$((96 + (4<<8))) KSPLIT=1 timeout 120 python tools/dbg4.py 1024 4096 16 ) > gpurun_out/trace_t.log 2>&1
cat gpurun_out/trace_t.log
