mkdir -p gpurun_out
export MQ_LIB=build_var/lib_dev.so
timeout 400 python tools/dbg_prefill.py > gpurun_out/prefill_dbg.log 2>&1
( MQ_DBG=$((96 + (5<<8))) NCH=40 timeout 120 python tools/dbg4.py 14336 4096 512 ) > gpurun_out/trace512.log 2>&1
cat gpurun_out/prefill_dbg.log; tail -45 gpurun_out/trace512.log
