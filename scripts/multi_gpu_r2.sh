python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench_n2_r2z.json 2> gpurun_out/bench_n2_r2z.err; echo n2 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/bench_n4_r2z.json 2> gpurun_out/bench_n4_r2z.err; echo n4 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_n4_ref_r2z.json 2> gpurun_out/bench_n4_ref_r2z.err; echo n4ref rc=$?
python -m pytest tests/test_gpu_multi.py -q > gpurun_out/pytest_multi4.txt 2>&1; echo multi rc=$?
