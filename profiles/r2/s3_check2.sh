# session 3: full GPU tests after the ring changes, ring cycle profile at the new defaults
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
PK_BUILD_DEFINES=-DAT_RING_PROF python -m paper_2511_13940_b200.build > /dev/null 2>&1
PK_LIB=paper_2511_13940_b200/libpk_DAT_RING_PROF.so python profiles/ring_prof.py > gpurun_out/ring_prof_s3.jsonl 2> gpurun_out/ring_prof_s3.err
