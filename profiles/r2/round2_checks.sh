python profiles/rs_precision.py --size 16384 > profiles/r2/rs_precision.jsonl 2> gpurun_out/rs_precision.err
python -m pytest tests/test_gpu_compat.py -q -x > gpurun_out/compat.log 2>&1; echo rc=$? >> gpurun_out/compat.log
cp profiles/r2/rs_precision.jsonl gpurun_out/
