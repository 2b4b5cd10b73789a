# quick loop: build, C4 stage times (optional options in $QS), then the full GPU suite
set -x
O=gpurun_out/${QO:-q}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
eval "timeout 600 python tools/stage_run.py C4 1.0 ${QS:-dict\(\)}" > $O/stage.log 2>&1; echo "stage rc $?"
cat $O/stage.log
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -15 $O/pytest.log; fi
