mkdir -p gpurun_out
( MQ_DBG=$((96 + (30<<8))) timeout 120 python tools/dbg4.py 14336 4096 16;
  MQ_DBG=$((96 + (2<<8))) timeout 120 python tools/dbg4.py 14336 4096 16;
  MQ_DBG=$((96 + (30<<8))) timeout 120 python tools/dbg4.py 28672 8192 16 ) > gpurun_out/trace2.log 2>&1
cat gpurun_out/trace2.log
