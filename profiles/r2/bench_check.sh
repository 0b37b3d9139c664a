# r2: bench N=1 (all legs) and the N=2 torchrun contract test (gloo plumbing on one GPU)
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo rc=$? >> gpurun_out/bench_n1.err
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x -k bench > gpurun_out/bench_n2_test.log 2>&1; echo rc=$? >> gpurun_out/bench_n2_test.log
PK_BENCH_DEVICE=0 PK_BENCH_BACKEND=gloo PK_BENCH_AR_MAX_BYTES=67108864 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --size 4096 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$? >> gpurun_out/bench_n2.err
