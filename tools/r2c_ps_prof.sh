# presplit k_split1<paired> in one device-resident launch: launch list + one full capture
set -x
mkdir -p gpurun_out/psp
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/psp/build.log 2>&1
: skip KMC_OPTS=x timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/psp/launches.csv python tools/profile_run.py C4 1.0 1 > gpurun_out/psp/l.log 2>&1; echo "list rc $?"
KMC_OPTS='dict(presplit=1)' timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_split1<\(bool\)1, \(bool\)1>" -c 1 -f -o gpurun_out/psp/full_pair python tools/profile_run.py C4 1.0 1 > gpurun_out/psp/f.log 2>&1; echo "full rc $?"
