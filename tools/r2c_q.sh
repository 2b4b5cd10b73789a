# quick: sampled/presplit tests + split tests + C4 stage times + e2e A/B
set -x
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q/build.log 2>&1
timeout 1200 python -m pytest tests/test_sampled.py tests/test_gpu_parity.py -m gpu -x -q -k "${QK:-sampled or presplit or split or forced or full_c4_exact}" > gpurun_out/q/pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/q/pytest.log
eval "timeout 600 python tools/stage_run.py C4 1.0 ${QS:-dict\(\)}" > gpurun_out/q/stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/q/stage.log
if [ -n "$QAB" ]; then eval "timeout 900 python tools/e2e_ab.py 1.0 3 $QAB" > gpurun_out/q/ab.log 2>&1; echo "ab rc $?"; cat gpurun_out/q/ab.log; fi
