python - <<'PY'
import torch, subprocess
PY
for e in "OUTDEV=cuda" "OUTDEV=cpu"; do echo "== $e"; for rep in 1 2; do env $e KMC_HOLD=1 timeout 300 python tools/pipe_probe.py 2>&1 | grep -v "^ " | grep -E "ms for|Error:" | head -1; done; done
