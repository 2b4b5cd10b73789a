# ncu full capture of the cluster kernel on C4 at 10% scale
set -x
python tools/cl_sweep.py C4 0.1 16 2>&1 | tail -3
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_clcount -c 1 -f -o gpurun_out/clc01 \
  python tools/profile_run.py C4 0.1 1 > gpurun_out/clc01.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/clc01.log
