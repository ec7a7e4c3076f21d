mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_hpass_block -c 1 \
  -o gpurun_out/prof_h1_hpass python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof_h1.log 2>&1; echo rc=$?
