# soak: the GPU suite three times back to back plus the fuzz sweep at 5x scale
for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/soak_$i.log 2>&1; echo rc=$? >> gpurun_out/soak_$i.log; done
PK_FUZZ_SCALE=5 timeout 1200 python -m pytest -x -q tests/test_gpu_fuzz.py > gpurun_out/soak_fuzz5.log 2>&1; echo rc=$? >> gpurun_out/soak_fuzz5.log
