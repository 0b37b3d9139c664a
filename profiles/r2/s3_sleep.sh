PK_BUILD_DEFINES=-DPK_EPI_SLEEP=0 python -m paper_2511_13940_b200.build > /dev/null 2>&1
python -m pytest -x -q tests/test_gpu_gemm_ops.py > gpurun_out/pytest_sleep.log 2>&1; echo rc=$? >> gpurun_out/pytest_sleep.log
for rep in 1 2 3; do for L in libpk.so libpk_DPK_EPI_SLEEP_0.so; do
  PK_LIB=paper_2511_13940_b200/$L SMS=148 REPS=1 OUT=/tmp/p.jsonl python profiles/gemm_sms_power.py | sed "s/^{/{\"lib\": \"$L\", /" >> gpurun_out/gemm_sleep_power.jsonl
done; done
SHAPES="16384 16384 16384;16384 16384 2048" bash profiles/gemm_cycles_ab.sh gpurun_out/gemm_sleep_cycles.csv paper_2511_13940_b200/libpk.so paper_2511_13940_b200/libpk_DPK_EPI_SLEEP_0.so
