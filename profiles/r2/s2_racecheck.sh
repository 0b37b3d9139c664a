mkdir -p gpurun_out/s2r
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2r/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/s2r/sanitizer_racecheck.log
timeout 600 python -m pytest -x -q tests/test_gpu_gemm_ops.py tests/test_gpu_grouped.py tests/test_gpu_moe.py > gpurun_out/s2r/pytest.log 2>&1; echo rc=$? >> gpurun_out/s2r/pytest.log
timeout 300 python bench.py --no-e2e --cpu-seconds 0.5 > gpurun_out/s2r/bench.json 2>/dev/null
