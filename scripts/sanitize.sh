mkdir -p gpurun_out
timeout 300 python scripts/sanitize.py 16 17 18 > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize.py 16 > gpurun_out/sanitize.log 2>&1; echo sanitize rc=$?
