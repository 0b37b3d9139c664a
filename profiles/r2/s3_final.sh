# session 3 captures on the final code (run from the repo root under gpurun)
set -u
OUT=gpurun_out/s3f
mkdir -p "$OUT"
python -m pytest tests -m gpu -x -q > "$OUT/pytest_all.log" 2>&1; echo rc=$? >> "$OUT/pytest_all.log"
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo smoke_rc=$? >> "$OUT/smoke.log"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_smoke.csv" python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/ncu_smoke.log" 2>&1; echo ncu_rc=$? >> "$OUT/ncu_smoke.log"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_bench.csv" python bench.py --steps 2 --warmup 1 > "$OUT/bench_under_ncu.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lcsc_gemm -c 1 \
  -o "$OUT/gemm16k" python bench.py --steps 1 --warmup 0 --no-e2e --no-baseline --cpu-seconds 0.5 > "$OUT/gemm16k_capture.log" 2>&1
ncu -i "$OUT/gemm16k.ncu-rep" --page raw --csv > "$OUT/gemm16k_raw.csv" 2>/dev/null
ncu -i "$OUT/gemm16k.ncu-rep" --page details --csv > "$OUT/gemm16k_details.csv" 2>/dev/null
SQ=16384 SKV=16384 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn2_fwd -s 1 -c 1 \
  -o "$OUT/attn_pair16k" python profiles/attn_once.py > "$OUT/attn_pair_capture.log" 2>&1
ncu -i "$OUT/attn_pair16k.ncu-rep" --page raw --csv > "$OUT/attn_pair16k_raw.csv" 2>/dev/null
ncu -i "$OUT/attn_pair16k.ncu-rep" --page details --csv > "$OUT/attn_pair16k_details.csv" 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 \
  -o "$OUT/attn_rank" python profiles/attn_once.py > "$OUT/attn_capture.log" 2>&1
ncu -i "$OUT/attn_rank.ncu-rep" --page raw --csv > "$OUT/attn_rank_raw.csv" 2>/dev/null
ncu -i "$OUT/attn_rank.ncu-rep" --page details --csv > "$OUT/attn_rank_details.csv" 2>/dev/null
timeout 300 ncu --clock-control none -k regex:"moe|grp|lcsc" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python profiles/moe_once.py > "$OUT/moe_launches.csv" 2>&1
rm -f "$OUT"/*.ncu-rep
for i in 1 2; do timeout 600 python bench.py > "$OUT/bench_$i.json" 2> "$OUT/bench_$i.err"; done
timeout 900 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 1500 python bench_ops.py --out "$OUT/ops.jsonl" > "$OUT/ops.log" 2>&1
