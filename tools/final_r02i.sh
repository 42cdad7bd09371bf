# Round-2 closing pass on the final code: GPU tests, smoke, the default bench
# line, the reference arm, the bench launch list and one ncu --set full capture
# of the headline round kernel.  Writes gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py --csv gpurun_out/runs.csv > gpurun_out/bench.log 2>&1; echo BENCH_RC=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo REF_RC=$?; tail -c 300 gpurun_out/bench_ref.log
CONFIGS="headline" bash tools/profile_r02.sh > gpurun_out/profile.log 2>&1
ls gpurun_out | head -50
