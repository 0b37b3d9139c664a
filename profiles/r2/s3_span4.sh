WORLDS=2,4,8 SPANS=1,2 python profiles/ring_span_ab.py > gpurun_out/ring_span_ab3.jsonl 2> gpurun_out/ring_span_ab3.err
S=131072 WORLDS=8 REPS=2 SPANS=1,2 python profiles/ring_span_ab.py >> gpurun_out/ring_span_ab3.jsonl 2>> gpurun_out/ring_span_ab3.err
