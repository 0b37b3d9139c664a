for ns in 3 5; do PK_BUILD_DEFINES="-DAT2_STAGES=$ns" python -m paper_2511_13940_b200.build > /dev/null 2>&1; done
PK_LIB=paper_2511_13940_b200/libpk_DAT2_STAGES_5.so python -m pytest -x -q tests/test_gpu_ring_attention.py -k pair > gpurun_out/pytest_ns5.log 2>&1; echo rc=$? >> gpurun_out/pytest_ns5.log
SHAPES="16384 16384" bash profiles/attn_cycles_ab.sh gpurun_out/attn_ns_cycles.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DAT2_STAGES_3.so paper_2511_13940_b200/libpk_DAT2_STAGES_5.so
for rep in 1 2 3; do for L in libpk.so libpk_DAT2_STAGES_3.so libpk_DAT2_STAGES_5.so; do PK_LIB=paper_2511_13940_b200/$L REPS=1 SHAPES=16384x16384 python profiles/attn_pair_ab.py | grep '"pair"' | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/attn_ns_time.jsonl; done; done
