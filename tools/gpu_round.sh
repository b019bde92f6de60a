# Standard GPU evidence pass (run under gpurun): parity tests, quick timing,
# bench line, ncu launch list of the bench, one ncu --set full capture of K2.
# usage: bash tools/gpu_round.sh [tag] [skip-tests]
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
fi
timeout 300 python tools/quick_time.py > gpurun_out/quick_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/quick_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mixed_gemm -s 3 -c 2 \
   -o gpurun_out/prof_k2_$TAG -f python tools/ncu_target.py 14336 4096 16 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mixed_gemm -s 3 -c 1 \
   -o gpurun_out/prof_k2_m512_$TAG -f python tools/ncu_target.py 14336 4096 512 > gpurun_out/ncu_full512_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/quick_$TAG.log; tail -1 gpurun_out/bench_$TAG.log | cut -c1-2500
