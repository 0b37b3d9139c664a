PK_BUILD_DEFINES=-DAT_PROFILE python -m paper_2511_13940_b200.build > /dev/null 2>&1
PK_LIB=paper_2511_13940_b200/libpk_DAT_PROFILE.so PK_ATTN_PAIR=0 python profiles/attn_phase_prof.py > gpurun_out/attn_phase.jsonl 2> gpurun_out/attn_phase.err
