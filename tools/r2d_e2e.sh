# e2e check: the pinned-output tests, then the e2e breakdown (C4) and the full GPU suite
set -x
O=gpurun_out/${QO:-e2e}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_buffers or oversize or multipass_full or streamed" > $O/pt1.log 2>&1; echo "pytest-e2e rc $?"; tail -3 $O/pt1.log
timeout 600 python tools/e2e_breakdown.py 1.0 > $O/e2eb.log 2>&1; grep "iter\|stages\|legacy" $O/e2eb.log | tail -8
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest.log; fi
