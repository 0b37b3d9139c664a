# session 3: persistent CTA-pair attention kernel — parity, A/B vs single-CTA and cuDNN, MMA-only variants
python -m pytest tests/test_gpu_ring_attention.py -x -q -k "pair or single_rank or uneven" > gpurun_out/pytest_pair.log 2>&1; echo rc=$? >> gpurun_out/pytest_pair.log
python profiles/attn_pair_ab.py > gpurun_out/attn_pair_ab.jsonl 2> gpurun_out/attn_pair_ab.err
PK_BUILD_DEFINES=-DAT_MMA_ONLY python -m paper_2511_13940_b200.build > /dev/null 2>&1
PK_LIB=paper_2511_13940_b200/libpk_DAT_MMA_ONLY.so REPS=1 python profiles/attn_pair_ab.py > gpurun_out/attn_pair_mmaonly.jsonl 2> gpurun_out/attn_pair_mmaonly.err
