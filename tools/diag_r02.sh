# Diagnostic pass: raw per-tile stamps of the headline round + CUDA-core tile micro-benchmarks.
mkdir -p gpurun_out
timeout 120 python tools/trace_round.py --out gpurun_out/tr_default.json --raw gpurun_out/tr_default.npz > gpurun_out/tr_default.txt 2>&1; tail -1 gpurun_out/tr_default.txt
timeout 120 python tools/pool_micro.py > gpurun_out/pool_micro.txt 2>&1; cat gpurun_out/pool_micro.txt
for o in ${TRACE_OPTS:-}; do
  args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /')
  timeout 120 python tools/trace_round.py $args --out gpurun_out/tr_$o.json --raw gpurun_out/tr_$o.npz > gpurun_out/tr_$o.txt 2>&1 || echo "trace $o failed"
  echo "$o: $(tail -1 gpurun_out/tr_$o.txt)"
done
