# One gpurun iteration (debug aid): GPU parity tests, round traces for each
# TRACE_OPTS entry ("default" or comma-separated runtime options), optional bench ($BENCH args).
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for o in ${TRACE_OPTS:-default}; do
  if [ "$o" = default ]; then args=""; else args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /'); fi
  timeout 120 python tools/trace_round.py $args --out gpurun_out/tr_$o.json > gpurun_out/tr_$o.txt 2>&1 || echo "trace $o failed"
  tail -1 gpurun_out/tr_$o.txt
done
python tools/stage_summary.py gpurun_out/tr_*.json > gpurun_out/stages.txt 2>&1
if [ -n "$BENCH" ]; then timeout 600 python bench.py $BENCH > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log; fi
