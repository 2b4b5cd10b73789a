# bench line (reads the committed traffic json) + the k_sig full capture of the current instance
set -x
O=gpurun_out/last; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_sig<\(int\)1" -c 1 -f -o $O/full_k_sig \
  python tools/profile_run.py C4 1.0 1 > $O/full_k_sig.log 2>&1; echo "ncu k_sig rc $?"
