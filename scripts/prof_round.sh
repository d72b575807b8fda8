# One GPU box call: bench (default N=1), the launch list of the same bench command, and an
# ncu --set full capture of the K1 R>32 kernel. Outputs under gpurun_out/.
mkdir -p gpurun_out
set -x
timeout 300 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo bench rc=$?
timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/b3.json 2>/dev/null && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 120 python scripts/k1_time.py cfg5 2 && timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_plan_eval -s 3 -c 1 -o gpurun_out/k1_v11_kpl2 python scripts/k1_time.py cfg5 2 > gpurun_out/ncu_v11.log 2>&1; echo ncu rc=$?
