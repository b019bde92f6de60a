mkdir -p gpurun_out
TAG=${1:-s}
export MQ_LIB=${MQ_LIB:-paper_2412_14590_b200/libmixllm_b200.so}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mixed_gemm -s 3 -c 1 -o gpurun_out/src512_$TAG -f python tools/ncu_target.py 14336 4096 512 > gpurun_out/ncu512_$TAG.log 2>&1
tail -2 gpurun_out/ncu512_$TAG.log
