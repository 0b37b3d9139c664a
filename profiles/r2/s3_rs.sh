PK_BUILD_DEFINES=-DPK_PLAIN_TEMPTY=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
for rep in 1 2 3; do for L in libpk.so libpk_DPK_PLAIN_TEMPTY_0.so; do PK_LIB=paper_2511_13940_b200/$L python profiles/rs_local_ab.py >> gpurun_out/rs_local_ab.jsonl 2>>gpurun_out/rs_local_ab.err; done; done
