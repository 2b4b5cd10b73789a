# quick GPU check of the current build: selected parity tests, then a short bench
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/q_smoke.log 2>&1; tail -3 gpurun_out/q_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${QK:-cluster or forced or k_boundaries or count_parity or chunk_count}" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/q_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${QB:-} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc $?"
tail -3 gpurun_out/q_bench.err
