# Round-2 evidence run on one B200: bench (cfg5, cfg5_full, cfg4), the launch
# list of the cfg5 bench command, per-launch K1 instruction counts (cfg5,
# cfg5_full, cfg5_7b) and one ncu --set full capture of each cfg5 K1 launch.
# Usage: bash scripts/prof_round2.sh <tag>    (outputs under gpurun_out/)
tag=${1:-r2}
mkdir -p gpurun_out
M=smsp__thread_inst_executed.sum,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 400 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench rc=$?
timeout 400 python bench.py --config cfg5_full --steps 3 --warmup 3 --cpu-seconds 12 > gpurun_out/bench_full_$tag.json 2> gpurun_out/bench_full_$tag.err; echo bench_full rc=$?
timeout 400 python bench.py --config cfg4 --steps 5 --warmup 3 --cpu-seconds 4 > gpurun_out/bench_cfg4_$tag.json 2> gpurun_out/bench_cfg4_$tag.err; echo bench_cfg4 rc=$?
timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/b3_$tag.json 2>/dev/null && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_launch_$tag.log 2>&1; echo launches rc=$?
for c in cfg5 cfg5_full cfg5_7b; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/k1cnt_${c}_$tag.csv -k regex:k_plan_eval \
    --launch-skip 2 --launch-count 2 python scripts/k1_time.py $c 1 > /dev/null 2>&1; echo k1cnt $c rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plan_eval --launch-skip 2 --launch-count 2 \
  -o gpurun_out/k1_$tag python scripts/k1_time.py cfg5 1 > gpurun_out/ncu_k1_$tag.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/k1_$tag.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/k1_${tag}_source.csv 2>/dev/null
echo done
