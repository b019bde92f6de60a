mkdir -p gpurun_out
( for a in "130 4096 4096 0.1 fast" "129 1024 1024 0.1 fast" "200 1024 1024 0.1 fast" "256 1024 1024 0.1 fast" "160 4096 4096 0.1 fast" "250 4096 4096 0.2 fast" "1 1024 1024 0.1 fast" "3 300 256 0.5 fast" "16 64 128 0.5 fast"; do
    timeout 120 python tools/probe_parity.py $a 2>&1 | tail -1
  done ) > gpurun_out/probe2.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r1b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r1b.log
( for k in 0 1; do for s in "14336 4096 16" "4096 4096 16" "1024 4096 16" "28672 8192 16"; do KSPLIT=$k timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done; done ) > gpurun_out/dbg3b.log
cat gpurun_out/probe2.log; tail -3 gpurun_out/pytest_gpu_r1b.log; cat gpurun_out/dbg3b.log
