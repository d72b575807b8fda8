# round-end style check on one B200: GPU suite, smoke, default bench, reference arm
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.txt 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref rc=$?
