# Exact-path robustness check: config 1-B&B timing, the random search case whose
# trees are far past the node budget (bounded phase A + sequential fallback),
# the exact-path tests with every plan forced onto the sequential fallback
# (OSERVE_EXACT_WORK=0; thread-per-plan and warp-per-plan kernels), then the
# exact and random-problem suites.
timeout 300 python scripts/time_exact.py > gpurun_out/xf_time.txt 2>&1; echo time rc=$?
for m in thread warp; do
  OSERVE_EXACT_SEQ=$m OSERVE_DEBUG_EXACT=1 timeout 400 python scripts/search_case.py 1202 2 gpu > gpurun_out/xf_search_$m.txt 2>&1; echo search $m rc=$?
  OSERVE_EXACT_SEQ=$m OSERVE_EXACT_WORK=0 timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > gpurun_out/xf_forced_$m.txt 2>&1; echo forced $m rc=$?
done
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_random_rounds.py -q -x --durations=5 > gpurun_out/xf_pytest.txt 2>&1; echo pytest rc=$?
