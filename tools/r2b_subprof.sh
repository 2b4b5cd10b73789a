# ncu full capture of the two sub-signature kernels at C4 (large_path 4)
set -x
KMC_OPTS='dict(large_path=4)' timeout 300 python tools/profile_run.py C4 1.0 1 > gpurun_out/subprof_plain.log 2>&1; tail -2 gpurun_out/subprof_plain.log
KMC_OPTS='dict(large_path=4)' timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_sub -c 2 -f -o gpurun_out/subprof \
  python tools/profile_run.py C4 1.0 1 > gpurun_out/subprof.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/subprof.log
