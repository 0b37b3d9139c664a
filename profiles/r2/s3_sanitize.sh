mkdir -p gpurun_out/s3san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python profiles/ring_sanitize.py > gpurun_out/s3san/ring_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/s3san/ring_$tool.log
done
