# session 3: ring attention with intra-SM communicator warps vs dedicated comm CTAs
python -m pytest tests/test_gpu_ring_attention.py tests/test_gpu_full_size.py tests/test_gpu_graphs.py -x -q > gpurun_out/pytest_ring.log 2>&1; echo rc=$? >> gpurun_out/pytest_ring.log
python profiles/ring_sweep.py > gpurun_out/ring_sweep_s3.jsonl 2> gpurun_out/ring_sweep_s3.err
