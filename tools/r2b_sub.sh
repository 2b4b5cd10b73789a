# sub-signature large path: parity tests, then C4 stage times against the default path
set -x
timeout 900 python -m pytest tests/test_subsplit.py -x -q > gpurun_out/sub_pytest.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/sub_pytest.log
timeout 600 python tools/stage_run.py C4 1.0 'dict()' 'dict(large_path=4)' > gpurun_out/sub_stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/sub_stage.log | tail -5
