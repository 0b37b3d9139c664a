PK_BUILD_DEFINES=-DAT2_RELAXED_ARRIVE=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
PK_BUILD_DEFINES="-DAT_MMA_ONLY" python -m paper_2511_13940_b200.build > /dev/null 2>&1
python -m pytest -x -q tests/test_gpu_ring_attention.py -k pair > gpurun_out/pytest_pair2.log 2>&1; echo rc=$? >> gpurun_out/pytest_pair2.log
for L in libpk.so libpk_DAT2_RELAXED_ARRIVE_0.so libpk_DAT_MMA_ONLY.so; do
  PK_LIB=paper_2511_13940_b200/$L REPS=1 SHAPES=16384x16384,8192x65536 python profiles/attn_pair_ab.py | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/attn_pair2.jsonl 2>> gpurun_out/attn_pair2.err
done
