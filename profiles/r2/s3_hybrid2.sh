python -m pytest -x -q tests/test_gpu_gemm_ops.py tests/test_gpu_graphs.py tests/test_gpu_compat.py tests/test_gpu_full_size.py tests/test_gpu_tune.py tests/test_gpu_multiprocess.py > gpurun_out/pytest_hybrid2.log 2>&1; echo rc=$? >> gpurun_out/pytest_hybrid2.log
python bench_ops.py --only local --out gpurun_out/ops_local_s3.jsonl > gpurun_out/ops_local_s3.log 2>&1
