# sampled-edge fixtures from oracle/_ref on the GPU box's host (196 GB RAM, 16 cores)
mkdir -p gpurun_out/golden
free -g | head -2
timeout 2400 python tests/golden/make_scale_golden.py sample rmat:26:1 --threads 16 --heavy 1000 --uniform 30000 --out gpurun_out/golden > gpurun_out/golden/rmat26.log 2>&1; echo r26 rc=$?
tail -3 gpurun_out/golden/rmat26.log
ls -la gpurun_out/golden
