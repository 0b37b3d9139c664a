PK_BUILD_DEFINES=-DPK_PLAIN_TEMPTY=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
python -m pytest -x -q tests/test_gpu_gemm_ops.py tests/test_gpu_grouped.py tests/test_gpu_gemm_ar.py > gpurun_out/pytest_tempty.log 2>&1; echo rc=$? >> gpurun_out/pytest_tempty.log
bash profiles/gemm_cycles_ab.sh gpurun_out/gemm_tempty_cycles.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DPK_PLAIN_TEMPTY_0.so
