mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo BENCH_RC=$? >> gpurun_out/bench.log
tail -c 400 gpurun_out/bench.log
timeout 120 python tools/trace_round.py --out gpurun_out/tr_default.json > gpurun_out/tr_default.txt 2>&1; tail -2 gpurun_out/tr_default.txt
