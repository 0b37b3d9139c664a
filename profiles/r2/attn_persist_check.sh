mkdir -p gpurun_out/persist
timeout 600 python -m pytest -x -q tests/test_gpu_ring_attention.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py > gpurun_out/persist/pytest.log 2>&1; echo rc=$? >> gpurun_out/persist/pytest.log
O=gpurun_out/persist/power.jsonl; : > $O
for rep in 1 2; do
SDPA=$([ $rep = 1 ] && echo 1 || echo 0) timeout 300 python profiles/attn_power.py $O
PK_ATTN_NO_PERSIST=1 SDPA=0 timeout 300 python profiles/attn_power.py $O
done
timeout 600 python bench_ops.py --only attn --out gpurun_out/persist/ops_attn.jsonl > /dev/null 2>&1
