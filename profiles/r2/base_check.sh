set -u
mkdir -p gpurun_out/r2b
python -m pytest tests -m gpu -x -q > gpurun_out/r2b/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/r2b/pytest_all.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b/bench_n1.json 2> gpurun_out/r2b/bench_n1.err
timeout 600 python bench_ops.py --only attn --out gpurun_out/r2b/ops_attn.jsonl > /dev/null 2>&1
python -c "import torch; from torch.nn.attention import sdpa_kernel, SDPBackend; print(torch.backends.cudnn.version())" >> gpurun_out/r2b/env.txt 2>&1
