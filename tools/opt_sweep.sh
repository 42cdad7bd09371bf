# Headline round-trace A/B over runtime options (each twice)
for o in default ${OPTS}; do
  if [ "$o" = default ]; then args=""; else args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /'); fi
  for rep in 1 2; do
    timeout 120 python tools/trace_round.py $args --out gpurun_out/sw.json > gpurun_out/sw.txt 2>&1 || echo "$o failed"
    echo "$o: $(tail -1 gpurun_out/sw.txt)"
  done
done
