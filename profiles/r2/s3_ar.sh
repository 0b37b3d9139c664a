python -m pytest -x -q tests/test_gpu_gemm_ar.py tests/test_gpu_gemm_ops.py tests/test_gpu_graphs.py tests/test_gpu_compat.py tests/test_gpu_tune.py > gpurun_out/pytest_ar.log 2>&1; echo rc=$? >> gpurun_out/pytest_ar.log
python bench_ops.py --only local --out gpurun_out/ops_local_s3b.jsonl > gpurun_out/ops_local_s3b.log 2>&1
