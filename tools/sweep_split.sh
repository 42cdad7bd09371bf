# Headline round-trace A/B: split-K (full-width tiles split over K) vs narrowing
set +e
OPTS=${OPTS:-"split_k=1 split_k=1,max_splits=2 split_k=1,max_splits=3 split_k=1,split_min_kb=16"}
for o in default $OPTS; do
  if [ "$o" = default ]; then args=""; else args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /'); fi
  for rep in 1 2; do
    f=gpurun_out/sw_${o}_${rep}
    timeout 120 python tools/trace_round.py $args --out $f.json > $f.txt 2>&1 || echo "$o failed"
    echo "$o: $(tail -1 $f.txt)"
  done
done
