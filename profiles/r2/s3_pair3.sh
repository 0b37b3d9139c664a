python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
bash profiles/attn_cycles_ab.sh gpurun_out/attn_pair_cycles.csv paper_2511_13940_b200/libpk.so cudnn
