#!/bin/bash
# Regenerate the profiles of one round on a B200 (run from the repo root under
# gpurun): the bench launch list, one full ncu capture of the headline GEMM
# kernel, the MoE kernel list and the per-op table.
#   gpurun --timeout 1800 -- 'bash profiles/capture.sh r1'
set -u
R=${1:-r1}
OUT=gpurun_out/$R
mkdir -p "$OUT"
# 1. every launch of a short bench run (cold-cache, serialised per-launch times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_bench.csv" python bench.py --steps 2 --warmup 1 > "$OUT/bench_under_ncu.log" 2>&1
# 2. one full capture of the LCSC GEMM kernel at 16384^3 (the AG-GEMM of the first step)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lcsc_gemm -c 1 \
  -o "$OUT/gemm16k" python bench.py --steps 1 --warmup 0 --no-e2e --no-baseline --cpu-seconds 0.5 > "$OUT/gemm16k_capture.log" 2>&1
ncu -i "$OUT/gemm16k.ncu-rep" --page raw --csv > "$OUT/gemm16k_raw.csv" 2>/dev/null
ncu -i "$OUT/gemm16k.ncu-rep" --page details --csv > "$OUT/gemm16k_details.csv" 2>/dev/null
# 3. MoE kernels (dispatch / grouped GEMM / combine) at the BASELINE shape
timeout 300 ncu --clock-control none -k regex:"moe|grp|lcsc" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python profiles/moe_once.py > "$OUT/moe_launches.csv" 2>&1
# 4. full captures of the attention rank step (n = 8, S = 32K) and the MoE dispatch kernel
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 \
  -o "$OUT/attn_rank" python profiles/attn_once.py > "$OUT/attn_capture.log" 2>&1
ncu -i "$OUT/attn_rank.ncu-rep" --page raw --csv > "$OUT/attn_rank_raw.csv" 2>/dev/null
ncu -i "$OUT/attn_rank.ncu-rep" --page details --csv > "$OUT/attn_rank_details.csv" 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_dispatch -s 1 -c 1 \
  -o "$OUT/moe_dispatch" python profiles/moe_once.py > "$OUT/moe_capture.log" 2>&1
ncu -i "$OUT/moe_dispatch.ncu-rep" --page raw --csv > "$OUT/moe_dispatch_raw.csv" 2>/dev/null
ncu -i "$OUT/moe_dispatch.ncu-rep" --page details --csv > "$OUT/moe_dispatch_details.csv" 2>/dev/null
# 5. the bench line itself (not under a profiler)
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
tail -1 "$OUT/bench.json"
