# full GPU suite + C4 stage times ($QS option dicts)
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/f_pytest.log
timeout 600 python tools/stage_run.py C4 1.0 ${QS:-'dict()'} > gpurun_out/f_stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/f_stage.log
