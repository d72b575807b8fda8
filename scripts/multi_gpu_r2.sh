# 2/4-GPU bench lines (library NCCL), the 4-GPU reference arm and the multi-GPU tests (gpurun --gpus 4)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench_n2_r2k.json 2> gpurun_out/bench_n2_r2k.err; echo n2 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/bench_n4_r2k.json 2> gpurun_out/bench_n4_r2k.err; echo n4 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_n4_ref_r2k.json 2> gpurun_out/bench_n4_ref_r2k.err; echo n4ref rc=$?
python -m pytest tests/test_gpu_multi.py -q > gpurun_out/pytest_multi4.txt 2>&1; echo multi rc=$?
timeout 300 oracle/_ref/dropin_test --devices 0,1,2,3 > gpurun_out/dropin_multi_r2k.txt 2>&1; echo dropin_multi rc=$?
