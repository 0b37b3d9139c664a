SHAPES="16384 16384;131072 16384" bash profiles/attn_cycles_ab.sh gpurun_out/attn_pair_cycles2.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk.so,PK_ATTN_PAIR=0 cudnn
