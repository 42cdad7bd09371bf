# One build->measure iteration: GPU tests (optional subset), CUDA-core tile micro-benchmarks, headline round trace.
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-600} python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 120 python tools/pool_micro.py > gpurun_out/pool_micro.txt 2>&1; cat gpurun_out/pool_micro.txt
timeout 120 python tools/trace_round.py --out gpurun_out/tr_default.json --raw gpurun_out/tr_default.npz > gpurun_out/tr_default.txt 2>&1; tail -1 gpurun_out/tr_default.txt
for o in ${TRACE_OPTS:-}; do
  args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /')
  timeout 120 python tools/trace_round.py $args --out gpurun_out/tr_$o.json --raw gpurun_out/tr_$o.npz > gpurun_out/tr_$o.txt 2>&1 || echo "trace $o failed"
  echo "$o: $(tail -1 gpurun_out/tr_$o.txt)"
done
if [ -n "$BENCH" ]; then timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo BENCH_RC=$?; tail -c 300 gpurun_out/bench.log; fi
