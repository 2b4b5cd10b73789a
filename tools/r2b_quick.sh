# quick check: selected parity tests ($QK) + C4 stage times for option dicts ($QS)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_subsplit.py -m gpu -x -q -k "${QK:-split or forced or count_parity or chunk or full_c4_exact or random_sweep or noncanonical}" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/q_pytest.log
timeout 600 python tools/stage_run.py C4 1.0 ${QS:-'dict()'} > gpurun_out/q_stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/q_stage.log
