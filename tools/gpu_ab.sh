# A/B timing of library variants on one box:
#   bash tools/gpu_ab.sh tag "ENV=.. lib" "lib2" ...   (AB_SET: quick_time.py argument)
mkdir -p gpurun_out
TAG=$1; shift
: > gpurun_out/ab_$TAG.log
for round in 1 2; do
for V in "$@"; do
  echo "== $V (round $round)" >> gpurun_out/ab_$TAG.log
  L=${V##* }; E=${V% *}; [ "$E" = "$V" ] && E=""
  env $E MQ_LIB=$L timeout 300 python tools/quick_time.py ${AB_SET:-prefill} >> gpurun_out/ab_$TAG.log 2>&1
done
done
cat gpurun_out/ab_$TAG.log
