# ncu full capture of the main C4 kernels (default path), one call
set -x
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_sig|k_split1|k_chunk_hash|k_rec_scatter|k_ord_scatter|k_ord_wsort" -c 9 -f -o gpurun_out/mainprof \
  python tools/profile_run.py C4 1.0 1 > gpurun_out/mainprof.log 2>&1; echo "ncu rc $?"
tail -2 gpurun_out/mainprof.log
