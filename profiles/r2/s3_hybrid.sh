python -m pytest -x -q tests/test_gpu_gemm_ops.py tests/test_gpu_graphs.py tests/test_gpu_compat.py > gpurun_out/pytest_hybrid.log 2>&1; echo rc=$? >> gpurun_out/pytest_hybrid.log
python profiles/ag_modes.py > gpurun_out/ag_modes.jsonl 2> gpurun_out/ag_modes.err
