python profiles/ring_span_ab.py > gpurun_out/ring_span_ab.jsonl 2> gpurun_out/ring_span_ab.err
S=131072 WORLDS=8 REPS=2 python profiles/ring_span_ab.py >> gpurun_out/ring_span_ab.jsonl 2>> gpurun_out/ring_span_ab.err
