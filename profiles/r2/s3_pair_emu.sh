for e in 0 2; do PK_BUILD_DEFINES="-DAT_EXP_EMU=$e" python -m paper_2511_13940_b200.build > /dev/null 2>&1; done
for rep in 1 2 3; do for L in libpk.so libpk_DAT_EXP_EMU_0.so libpk_DAT_EXP_EMU_2.so; do PK_LIB=paper_2511_13940_b200/$L REPS=1 SHAPES=16384x16384,16384x131072 python profiles/attn_pair_ab.py | grep '"pair"' | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/pair_emu_time.jsonl; done; done
