for d in "-DAT_PQ=4" "-DAT_EXP_EMU=0" "-DAT_EXP_EMU=2"; do PK_BUILD_DEFINES="$d" python -m paper_2511_13940_b200.build > /dev/null 2>&1; done
PK_LIB=paper_2511_13940_b200/libpk_DAT_PQ_4.so python -m pytest -x -q tests/test_gpu_ring_attention.py > gpurun_out/pytest_pq4.log 2>&1; echo rc=$? >> gpurun_out/pytest_pq4.log
bash profiles/attn_cycles_ab.sh gpurun_out/attn_pq_cycles.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DAT_PQ_4.so paper_2511_13940_b200/libpk_DAT_EXP_EMU_0.so paper_2511_13940_b200/libpk_DAT_EXP_EMU_2.so
