mkdir -p gpurun_out/sdpa
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x
F='regex:^((?!elementwise).)*$'
SQ=8192 SKV=65536 timeout 300 ncu --clock-control base --metrics $M -k "$F" -c 2 --csv python profiles/sdpa_once.py > gpurun_out/sdpa/ncu_sdpa.csv 2>&1
SQ=16384 SKV=16384 timeout 300 ncu --clock-control base --metrics $M -k "$F" -c 2 --csv python profiles/sdpa_once.py > gpurun_out/sdpa/ncu_sdpa_16k.csv 2>&1
