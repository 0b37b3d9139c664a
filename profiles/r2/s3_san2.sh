mkdir -p gpurun_out/s3san2
SCHEDS=default timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python profiles/hybrid_sanitize.py > gpurun_out/s3san2/default_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/s3san2/default_racecheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3san2/smoke_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/s3san2/smoke_racecheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3san2/smoke_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/s3san2/smoke_memcheck.log
