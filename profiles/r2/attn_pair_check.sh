mkdir -p gpurun_out/pair
O=gpurun_out/pair/power.jsonl; : > $O
SDPA=0 timeout 300 python profiles/attn_power.py $O
PK_ATTN_PAIR=1 SDPA=0 timeout 300 python profiles/attn_power.py $O
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_wait,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed
SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --metrics $M -k regex:attn -s 1 -c 1 --csv python profiles/attn_once.py > gpurun_out/pair/ncu_single.csv 2>&1
PK_ATTN_PAIR=1 SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --metrics $M -k regex:attn -s 1 -c 1 --csv python profiles/attn_once.py > gpurun_out/pair/ncu_pair.csv 2>&1
PK_LIB=paper_2511_13940_b200/libpk_DAT_CW_1__DAT_MMA_ONLY.so SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --metrics $M -k regex:attn -s 1 -c 1 --csv python profiles/attn_once.py > gpurun_out/pair/ncu_mmaonly.csv 2>&1
