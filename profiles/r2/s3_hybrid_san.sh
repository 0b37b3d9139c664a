mkdir -p gpurun_out/s3san
python profiles/hybrid_sanitize.py > gpurun_out/s3san/hybrid_plain.log 2>&1; echo "rc=$?" >> gpurun_out/s3san/hybrid_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python profiles/hybrid_sanitize.py > gpurun_out/s3san/hybrid_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/s3san/hybrid_$tool.log
done
