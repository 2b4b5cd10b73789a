set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; tail -2 gpurun_out/b_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/b_pytest.log
timeout 600 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc $?"
tail -3 gpurun_out/b_bench.err
