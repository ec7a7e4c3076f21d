# Fast iteration: GPU parity (incl. slow RMAT-20 sample) + a short bench.  Usage: bash scripts/quick_gpu.sh <tag> [pytest -k expr]
TAG=${1:-q}
mkdir -p gpurun_out
K=${2:+-k "$2"}
timeout 900 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?
python - <<'P'
import json,sys,glob,os
tag=os.environ.get('TAG')
P
tail -c 1500 gpurun_out/bench_${TAG}.log
