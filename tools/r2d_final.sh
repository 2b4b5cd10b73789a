# final evidence of the session: smoke, the full GPU suite, then the profile suite (bench line,
# ncu launch list, full captures of the three top kernels)
set -x
mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/fin/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/fin/pytest.log
OUT=gpurun_out/fin bash tools/r2_profile_suite.sh
