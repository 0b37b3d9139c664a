python -m pytest -x -q tests/test_gpu_ring_attention.py > gpurun_out/pytest_ab2.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab2.log
bash profiles/attn_cycles_ab.sh gpurun_out/attn_ab2_cycles.csv paper_2511_13940_b200/libpk_s3start_attn.so paper_2511_13940_b200/libpk.so cudnn
