# attention energy / cycles per call across builds, then ncu cycle + stall metrics for CW=1 vs CW=2
set -u
mkdir -p gpurun_out/ap
L=paper_2511_13940_b200
O=gpurun_out/ap/attn_power.jsonl
: > $O
for rep in 1 2; do
for lib in libpk_DAT_CW_1.so libpk.so libpk_DAT_CW_1__DAT_MMA_ONLY.so libpk_DAT_CW_1__DAT_EXP_EMU_0.so libpk_DAT_CW_1__DAT_EXP_EMU_2.so; do
  SDPA=$([ $lib = libpk_DAT_CW_1.so ] && echo 1 || echo 0) PK_LIB=$L/$lib timeout 300 python profiles/attn_power.py $O 2>> gpurun_out/ap/err.log
done
done
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_active.avg,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_math_pipe_throttle
for lib in libpk_DAT_CW_1.so libpk.so libpk_DAT_CW_1__DAT_MMA_ONLY.so; do
  PK_LIB=$L/$lib SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --metrics $M -k regex:attn_fwd -s 1 -c 1 --csv python profiles/attn_once.py > gpurun_out/ap/ncu_$lib.csv 2>&1
  PK_LIB=$L/$lib SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --section WarpStateStats -k regex:attn_fwd -s 1 -c 1 --csv --page details python profiles/attn_once.py > gpurun_out/ap/ncu_stall_$lib.csv 2>&1
done
