mkdir -p gpurun_out
( MQ_LIB=build_var/lib_dev.so MQ_DBG=$((96 + (5<<8) + ${EXTRA_DBG:-0})) NCH=${NCH:-40} timeout 120 python tools/dbg4.py ${SHAPE:-14336 4096 512} ) > gpurun_out/trace512${TAG}.log 2>&1
grep -E "^(1[6-9]|2[0-9]) |event|CTA" gpurun_out/trace512${TAG}.log
