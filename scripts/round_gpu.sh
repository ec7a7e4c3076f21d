# One gpurun call: smoke, GPU parity tests, bench (N=1), ncu launch list + full captures.
# Usage: bash scripts/round_gpu.sh <tag> [noprof]
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi -L; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo bench rc=$?
tail -c 2500 gpurun_out/bench_${TAG}.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo benchref rc=$?
timeout 600 python bench.py --graph ba --steps 3 --warmup 3 > gpurun_out/bench_ba_${TAG}.log 2>&1; echo bench_ba rc=$?
[ "$2" = "noprof" ] || bash scripts/profile.sh ${TAG}
