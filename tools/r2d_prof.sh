# full captures (source level) of the three top kernels, one C4 call each
set -x
OUT=${OUT:-gpurun_out/dp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_sig<\(int\)1" -c 1 -f -o $OUT/full_k_sig \
  python tools/profile_run.py C4 1.0 1 > $OUT/full_k_sig.log 2>&1; echo "ncu k_sig rc $?"
for kr in k_split1 k_chunk_hash; do
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$kr -c 1 -f -o $OUT/full_$kr \
    python tools/profile_run.py C4 1.0 1 > $OUT/full_$kr.log 2>&1; echo "ncu $kr rc $?"
done
ls -la $OUT
