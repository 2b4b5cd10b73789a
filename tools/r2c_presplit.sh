# presplit: parity tests + e2e A/B + device-resident stage times
set -x
mkdir -p gpurun_out/ps
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ps/build.log 2>&1
timeout 1200 python -m pytest tests/test_sampled.py -m gpu -x -q > gpurun_out/ps/pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/ps/pytest.log
timeout 900 python tools/e2e_ab.py 1.0 3 'dict(presplit=2)' 'dict()' > gpurun_out/ps/ab.log 2>&1; echo "ab rc $?"
cat gpurun_out/ps/ab.log
timeout 600 python tools/stage_run.py C4 1.0 'dict()' 'dict(presplit=1)' > gpurun_out/ps/stage.log 2>&1; echo "stage rc $?"
cat gpurun_out/ps/stage.log
