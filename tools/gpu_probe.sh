mkdir -p gpurun_out
( for a in "130 4096 4096 0.1 fast" "130 4096 4096 0.1 fast 128 1" "130 4096 4096 0.1 exact" "130 4096 4096 0.1 fast 64" \
           "129 1024 1024 0.1 fast" "200 1024 1024 0.1 fast" "257 1024 1024 0.1 fast" "256 1024 1024 0.1 fast" "130 1024 1024 0.0 fast" "130 1024 1024 1.0 fast"; do
    timeout 120 python tools/probe_parity.py $a 2>&1 | tail -1
  done ) > gpurun_out/probe.log
( for d in 0 1 2 4 6 7; do
    for s in "14336 4096 16" "4096 4096 16" "1024 4096 16"; do MQ_DBG=$d timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done
  done ) > gpurun_out/dbg3.log
( for s in "14336 4096 16" "4096 4096 16"; do MQ_DBG=96 timeout 120 python tools/dbg4.py $s 2>&1; done ) > gpurun_out/dbg4.log
cat gpurun_out/probe.log gpurun_out/dbg3.log
