# Config-2 K1 counters (the 16-lane-group kernel of the config-4 windows): CUDA-event timing, then an ncu --metrics pass
M=smsp__thread_inst_executed.sum,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,smsp__thread_inst_executed_per_inst_executed.ratio,sm__cycles_active.avg
timeout 120 python scripts/k1_time.py cfg2 3 > gpurun_out/cfg2_k1t.txt 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/cfg2_k1cnt.csv python scripts/k1_time.py cfg2 1 > /dev/null 2>&1; echo rc=$?
