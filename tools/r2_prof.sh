# ncu full capture of one kernel (regex $KREG) in one kmc_count call on $CFG at $SCALE
set -x
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:${KREG} -c 1 -f -o gpurun_out/${OUT:-prof} \
  python tools/profile_run.py ${CFG:-C4} ${SCALE:-1.0} 1 > gpurun_out/${OUT:-prof}.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/${OUT:-prof}.log
