# One GPU box call: bench (default N=1), the launch list of the same bench command, and
# ncu --set full captures of both K1 kernels (R <= 32 and R > 32 buckets) of config 5.
# Usage: bash scripts/prof_round.sh <tag>     (outputs under gpurun_out/)
tag=${1:-r1}
mkdir -p gpurun_out
set -x
timeout 300 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench rc=$?
timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/b3_$tag.json 2>/dev/null && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_launch_$tag.log 2>&1; echo launches rc=$?
timeout 120 python scripts/k1_time.py cfg5 2 && \
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_plan_eval -s 2 -c 2 \
  -o gpurun_out/k1_$tag python scripts/k1_time.py cfg5 2 > gpurun_out/ncu_k1_$tag.log 2>&1; echo ncu rc=$?
