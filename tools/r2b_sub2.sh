set -x
timeout 900 python -m pytest tests/test_subsplit.py -x -q > gpurun_out/sub_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/sub_pytest.log
timeout 600 python tools/stage_run.py C4 1.0 'dict(large_path=4)' > gpurun_out/sub_stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/sub_stage.log | tail -3
KMC_OPTS='dict(large_path=4)' timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_sub(split|count)" -c 2 -f -o gpurun_out/subprof \
  python tools/profile_run.py C4 1.0 1 > gpurun_out/subprof.log 2>&1; echo "ncu rc $?"
