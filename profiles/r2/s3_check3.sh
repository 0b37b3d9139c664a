python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all3.log 2>&1; echo rc=$? >> gpurun_out/pytest_all3.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke3.log
python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$? >> gpurun_out/bench3.err
