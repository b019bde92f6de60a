mkdir -p gpurun_out
( for d in 0 8; do for np in 0 1; do for s in "14336 4096 16" "4096 4096 16" "1024 4096 16"; do
   MQ_DBG=$d NOPDL=$np timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done; done; done
  for k in 1 2 4 8; do KSPLIT=$k timeout 120 python tools/dbg3.py 1024 4096 16 2>&1 | tail -1; done
  MQ_DBG=$((96 + (4<<8))) timeout 120 python tools/dbg4.py 1024 4096 16 ) > gpurun_out/floor.log 2>&1
cat gpurun_out/floor.log
