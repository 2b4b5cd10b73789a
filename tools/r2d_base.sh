# round-2 session-3 baseline: smoke, full GPU suite, full bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/d
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/d/smoke.log 2>&1; echo "smoke rc $?"
timeout 600 python bench.py > gpurun_out/d/bench.json 2> gpurun_out/d/bench.err; echo "bench rc $?"
cat gpurun_out/d/bench.json | head -c 600
timeout 600 python tools/stage_run.py C4 1.0 > gpurun_out/d/stage.log 2>&1; cat gpurun_out/d/stage.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/d/pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/d/pytest.log
