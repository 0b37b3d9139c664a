# r2 checks: multi-process tests (same GPU), N=2 bench over gloo on one GPU, loopback calibration
python -m pytest tests/test_gpu_multiprocess.py -q -x > gpurun_out/mp_tests.log 2>&1; echo rc=$? >> gpurun_out/mp_tests.log
PK_BENCH_DEVICE=0 PK_BENCH_BACKEND=gloo PK_BENCH_AR_MAX_BYTES=67108864 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --size 4096 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$? >> gpurun_out/bench_n2.err
python -m paper_2511_13940_b200.mechanisms --out gpurun_out/mech_loopback.json > /dev/null 2> gpurun_out/mech.err; echo rc=$? >> gpurun_out/mech.err
