# ncu evidence for the bench workload (one GPU).  Usage: bash scripts/profile.sh <tag> [scale]
set -x
TAG=${1:-r1}
SCALE=${2:-20}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --scale $SCALE"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $B > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
# dominant kernels: dense-window cycles, large/small block H-pass (count + sums)
for K in k_cycle_block k_hpass_block; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -c 3 \
      -o gpurun_out/prof_${TAG}_${K} $B > gpurun_out/prof_${TAG}_${K}.log 2>&1; echo $K rc=$?
done
