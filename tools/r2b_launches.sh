# stage times + ncu launch list (per-kernel durations) of one C4 call
set -x
timeout 600 python tools/stage_run.py C4 1.0 ${QS:-'dict()'} > gpurun_out/l_stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/l_stage.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches.csv \
  python tools/profile_run.py C4 1.0 1 > gpurun_out/l_ncu.log 2>&1; echo "ncu rc $?"
