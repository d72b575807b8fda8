# exact-path check: GPU parity tests that take the B&B path, then timings (old vs device-built frontier)
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_gpu_edge.py -q 2>&1 | tail -3
for bfs in 0 1; do
  echo "== BFS=$bfs"
  OSERVE_EXACT_BFS=$bfs timeout 300 python -m pytest tests/test_gpu_exact.py -q 2>&1 | tail -1
  OSERVE_EXACT_BFS=$bfs OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | tail -14
done
