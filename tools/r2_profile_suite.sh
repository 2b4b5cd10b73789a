# Round-2 evidence on one B200: bench line, ncu launch list of the bench command, full captures
set -x
OUT=${OUT:-gpurun_out/r2p}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
  --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sort-path > $OUT/ncu_bench.log 2>&1; echo "ncu list rc $?"
# k_sig: the scatter pass (k_sig<1>), not the sample pass (k_sig<0>)
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_sig<\(int\)1" -c 1 -f -o $OUT/full_k_sig \
  python tools/profile_run.py C4 1.0 1 > $OUT/full_k_sig.log 2>&1; echo "ncu k_sig rc $?"
for kr in k_split1 k_chunk_hash; do
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$kr -c 1 -f -o $OUT/full_$kr \
    python tools/profile_run.py C4 1.0 1 > $OUT/full_$kr.log 2>&1; echo "ncu $kr rc $?"
done
