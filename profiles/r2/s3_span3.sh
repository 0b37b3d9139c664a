python -m pytest tests/test_gpu_ring_attention.py tests/test_gpu_graphs.py tests/test_gpu_full_size.py -x -q > gpurun_out/pytest_span3.log 2>&1; echo rc=$? >> gpurun_out/pytest_span3.log
WORLDS=4,8 SPANS=1,2,3 python profiles/ring_span_ab.py > gpurun_out/ring_span_ab2.jsonl 2> gpurun_out/ring_span_ab2.err
S=131072 WORLDS=8 REPS=2 SPANS=1,2 python profiles/ring_span_ab.py >> gpurun_out/ring_span_ab2.jsonl 2>> gpurun_out/ring_span_ab2.err
PK_BUILD_DEFINES=-DAT_RING_PROF python -m paper_2511_13940_b200.build > /dev/null 2>&1
PK_LIB=paper_2511_13940_b200/libpk_DAT_RING_PROF.so python profiles/ring_prof.py > gpurun_out/ring_prof_s3b.jsonl 2> gpurun_out/ring_prof_s3b.err
