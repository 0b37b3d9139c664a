PK_BUILD_DEFINES=-DAT_RING_REGCOPY=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
python -m pytest -x -q tests/test_gpu_ring_attention.py tests/test_gpu_graphs.py > gpurun_out/pytest_regcopy.log 2>&1; echo rc=$? >> gpurun_out/pytest_regcopy.log
for L in libpk.so libpk_DAT_RING_REGCOPY_0.so; do PK_LIB=paper_2511_13940_b200/$L WORLDS=4,8 SPANS=1,2 REPS=4 python profiles/ring_span_ab.py | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/ring_regcopy.jsonl 2>> gpurun_out/ring_regcopy.err; done
for L in libpk_DAT_RING_REGCOPY_0.so libpk.so; do PK_LIB=paper_2511_13940_b200/$L WORLDS=8 SPANS=2 REPS=4 python profiles/ring_span_ab.py | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/ring_regcopy.jsonl 2>> gpurun_out/ring_regcopy.err; done
