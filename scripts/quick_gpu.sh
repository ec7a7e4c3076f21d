# Fast iteration: GPU parity (incl. slow RMAT-20 sample) + a short bench.  Usage: bash scripts/quick_gpu.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?
tail -c 1500 gpurun_out/bench_${TAG}.log
echo; tail -1 gpurun_out/pytest_${TAG}.log
