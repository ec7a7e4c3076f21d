set -x
mkdir -p gpurun_out
nvidia-smi -L; nproc
timeout 300 python scripts/sanitize.py 16 18 > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.log 2>&1; echo bench rc=$?
