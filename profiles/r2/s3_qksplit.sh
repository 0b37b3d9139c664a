PK_BUILD_DEFINES=-DAT_QK_SPLIT=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
python -m pytest -x -q tests/test_gpu_ring_attention.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py tests/test_gpu_full_size.py > gpurun_out/pytest_qksplit.log 2>&1; echo rc=$? >> gpurun_out/pytest_qksplit.log
bash profiles/attn_cycles_ab.sh gpurun_out/attn_qksplit_cycles.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DAT_QK_SPLIT_0.so
for rep in 1 2; do for L in libpk.so libpk_DAT_QK_SPLIT_0.so; do PK_LIB=paper_2511_13940_b200/$L REPS=1 python profiles/attn_pair_ab.py | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/attn_qksplit_time.jsonl; done; done
