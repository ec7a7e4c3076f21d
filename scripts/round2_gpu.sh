# Round-2 evidence in one gpurun call: smoke, GPU tests, bench lines (RMAT-20
# default incl. e2e variants, reference arm, BA configs[2], RMAT-24, RMAT-26),
# ncu launch list + DRAM traffic of the dominant kernel per workload, full ncu
# captures at RMAT-20.   Usage: bash scripts/round2_gpu.sh <tag>
TAG=${1:-r2f}
O=gpurun_out
mkdir -p $O
nvidia-smi -L; free -g | head -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_${TAG}.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $O/pytest_${TAG}.log 2>&1; echo pytest rc=$?; tail -25 $O/pytest_${TAG}.log
timeout 900 python bench.py > $O/bench_${TAG}.log 2>&1; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_${TAG}.log 2>&1; echo ref rc=$?
timeout 900 python bench.py --graph ba --steps 5 --warmup 3 > $O/bench_ba_${TAG}.log 2>&1; echo ba rc=$?
timeout 1500 python bench.py --scale 24 --steps 3 --warmup 3 --e2e-steps 2 --e2e-warmup 1 > $O/bench_s24_${TAG}.log 2>&1; echo s24 rc=$?
timeout 2400 python bench.py --scale 26 --steps 1 --warmup 3 --e2e-steps 1 --e2e-warmup 1 --no-cpu-baseline > $O/bench_s26_${TAG}.log 2>&1; echo s26 rc=$?
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${TAG}.csv $B > /dev/null 2>&1; echo launches rc=$?
for K in k_cycle_block k_hpass_block; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -c 1 -o $O/prof_${TAG}_${K} $B > /dev/null 2>&1; echo $K rc=$?
done
for W in "--graph ba" "--scale 24" "--scale 26"; do
  N=$(echo $W | tr -d ' -')
  timeout 1800 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:"k_cycle_block|k_hpass_block" --log-file $O/traffic_${TAG}_${N}.csv $B $W > /dev/null 2>&1; echo traffic $N rc=$?
done
