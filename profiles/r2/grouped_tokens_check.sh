# grouped GEMM token tiles (EPI_TOKENS_T) vs 256-row padded tiles (PK_GROUPED_PADDED=1)
mkdir -p gpurun_out/gt
timeout 600 python -m pytest -x -q tests/test_gpu_grouped.py tests/test_gpu_moe.py tests/test_gpu_edges.py > gpurun_out/gt/pytest.log 2>&1; echo rc=$? >> gpurun_out/gt/pytest.log
for rep in 1 2; do
timeout 300 python bench_ops.py --only moe --out gpurun_out/gt/moe_tokens_$rep.jsonl > /dev/null 2>&1
PK_GROUPED_PADDED=1 timeout 300 python bench_ops.py --only moe --out gpurun_out/gt/moe_padded_$rep.jsonl > /dev/null 2>&1
done
