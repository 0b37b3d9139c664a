# attention with two softmax warps per quadrant (AT_CW=2, libpk.so) vs one (libpk_DAT_CW_1.so)
set -u
mkdir -p gpurun_out/cw
timeout 600 python -m pytest -x -q tests/test_gpu_ring_attention.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py > gpurun_out/cw/pytest_attn.log 2>&1; echo rc=$? >> gpurun_out/cw/pytest_attn.log
tail -2 gpurun_out/cw/pytest_attn.log
timeout 900 bash profiles/attn_lib_ab.sh paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DAT_CW_1.so gpurun_out/cw/attn_ab.jsonl
