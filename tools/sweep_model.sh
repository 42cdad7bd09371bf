# Round-trace A/B of runtime options on one model config: MODEL, BATCH, TENANTS, OPTS
for o in default ${OPTS}; do
  if [ "$o" = default ]; then args=""; else args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /'); fi
  for rep in 1 2; do
    timeout 120 python tools/trace_round.py --model ${MODEL:-resnet50} --batch ${BATCH:-8} --tenants ${TENANTS:-4} $args > gpurun_out/swm.txt 2>&1 || echo "$o failed"
    echo "$MODEL b$BATCH $o: $(tail -1 gpurun_out/swm.txt)"
  done
done
