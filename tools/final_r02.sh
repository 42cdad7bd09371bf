# Round-2 final measurement pass: GPU tests, smoke, the default bench line,
# the profiling pass (launch list + ncu --set full per config), staged
# CUDA-core tile micro captures, headline round trace.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py --csv gpurun_out/runs.csv > gpurun_out/bench.log 2>&1; echo BENCH_RC=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo REF_RC=$?; tail -c 300 gpurun_out/bench_ref.log
bash tools/profile_r02.sh > gpurun_out/profile.log 2>&1
bash tools/ncu_pool.sh maxpool112; bash tools/ncu_pool.sh dw56
timeout 120 python tools/pool_micro.py > gpurun_out/pool_micro.txt 2>&1
timeout 120 python tools/trace_round.py --out gpurun_out/tr_default.json --raw gpurun_out/tr_default.npz > gpurun_out/tr_default.txt 2>&1
ls gpurun_out | head -50
