# ncu --set full of one kernel on the bench workload.  Usage: bash scripts/prof_one.sh <tag> <kernel-regex> [scale]
TAG=$1; K=$2; SCALE=${3:-20}
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
  -o gpurun_out/prof_${TAG}_${K} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --scale $SCALE \
  > gpurun_out/prof_${TAG}_${K}.log 2>&1; echo $K rc=$?
