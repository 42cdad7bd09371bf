set +e
for m in resnet50 mix bert; do
for o in default narrow_min_tiles=16 narrow_min_tiles=24 narrow_min_tiles=28 narrow_min_tiles=32 narrow_min_tiles=48; do
  if [ "$o" = default ]; then args=""; else args="--opt $o"; fi
  b=8; [ $m = resnet50 ] || b=4
  t=4; [ $m = bert ] && t=16
  r=""
  for rep in 1 2; do
    r="$r $(timeout 120 python tools/trace_round.py --model $m --tenants $t --batch $b $args 2>&1 | tail -1 | awk '{print $3}')"
  done
  echo "$m $o:$r"
done
done
