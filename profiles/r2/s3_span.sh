# session 3: ring unit span (2P stage slots) — parity and the n = 2/4/8 sweep
python -m pytest tests/test_gpu_ring_attention.py -x -q > gpurun_out/pytest_span.log 2>&1; echo rc=$? >> gpurun_out/pytest_span.log
SPANS=2,4 python profiles/ring_sweep.py > gpurun_out/ring_sweep_span.jsonl 2> gpurun_out/ring_sweep_span.err
