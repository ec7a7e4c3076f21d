# ncu launch list (gpu__time_duration per kernel) of one bench step.  Usage: bash scripts/launches.sh <tag> [scale]
TAG=$1; SCALE=${2:-20}
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --scale $SCALE \
  > gpurun_out/launches_${TAG}.log 2>&1; echo launches rc=$?
python scripts/launch_summary.py gpurun_out/launches_${TAG}.csv | head -14
