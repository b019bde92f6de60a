mkdir -p gpurun_out
timeout 600 python tools/dbg_matrix.py > gpurun_out/dbg_matrix.log 2>&1
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device python tools/dbg_matrix.py one 16 512 256 0.1 exact 128 16 > gpurun_out/sanitizer.log 2>&1
head -c 6000 gpurun_out/sanitizer.log
cat gpurun_out/dbg_matrix.log
