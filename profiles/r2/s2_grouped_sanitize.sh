mkdir -p gpurun_out/s2g
timeout 600 python -m pytest -x -q tests/test_gpu_grouped.py > gpurun_out/s2g/pytest_grouped.log 2>&1; echo rc=$? >> gpurun_out/s2g/pytest_grouped.log
# one full capture of the token-tile grouped GEMM (the first lcsc launch of moe_once.py is the planned GEMM1)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lcsc_gemm -s 0 -c 1 \
  -o gpurun_out/s2g/grouped_tokens python profiles/moe_once.py > gpurun_out/s2g/grouped_capture.log 2>&1
ncu -i gpurun_out/s2g/grouped_tokens.ncu-rep --page raw --csv > gpurun_out/s2g/grouped_tokens_raw.csv 2>/dev/null
ncu -i gpurun_out/s2g/grouped_tokens.ncu-rep --page details --csv > gpurun_out/s2g/grouped_tokens_details.csv 2>/dev/null
rm -f gpurun_out/s2g/*.ncu-rep
# compute-sanitizer over the world-1 smoke (every kernel family once)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2g/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/s2g/sanitizer_$tool.log
done
