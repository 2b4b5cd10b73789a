# build variants (KMC_NVCC_EXTRA flags, ';'-separated in $VARS) and time C4 stages for each
O=gpurun_out/${QO:-sw}
mkdir -p $O
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  KMC_NVCC_EXTRA="$v" python -m paper_1407_1507_b200.build --force > $O/build.log 2>&1 || { echo "build failed: $v"; tail -5 $O/build.log; continue; }
  echo "== $v"; timeout 300 python tools/stage_run.py C4 1.0 2>&1 | tail -1
done
