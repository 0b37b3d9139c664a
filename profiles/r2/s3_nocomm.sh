PK_BUILD_DEFINES=-DAT_RING_NOCOMM python -m paper_2511_13940_b200.build > /dev/null 2>&1
WORLDS=8 SPANS=1,2,8 REPS=3 python profiles/ring_span_ab.py > gpurun_out/ring_nocomm.jsonl 2> gpurun_out/ring_nocomm.err
PK_LIB=paper_2511_13940_b200/libpk_DAT_RING_NOCOMM.so WORLDS=8 SPANS=1,2,8 REPS=3 python profiles/ring_span_ab.py >> gpurun_out/ring_nocomm.jsonl 2>> gpurun_out/ring_nocomm.err
