# compute-sanitizer memcheck of the counting kernels on small graphs (one GPU).
mkdir -p gpurun_out
timeout 300 python scripts/sanitize.py 16 17 18 > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize.py 13 ba:20000:6 > gpurun_out/sanitize.log 2>&1; echo sanitize rc=$?
GL_SPARSE_BIG=all timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize.py ba:60000:6 recut > gpurun_out/sanitize_sparse.log 2>&1; echo sanitize_sparse rc=$?
