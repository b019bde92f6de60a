mkdir -p gpurun_out
for v in g4n8 g2n12 g1n16; do
  for k in 0 1; do for s in "14336 4096 16" "4096 4096 16" "1024 4096 16" "28672 8192 16"; do
    echo -n "$v "; MQ_LIB=build_var/lib_$v.so KSPLIT=$k timeout 120 python tools/dbg3.py $s 2>&1 | tail -1; done; done
done > gpurun_out/var.log 2>&1
cat gpurun_out/var.log
