set +e
for v in new old new old; do
  if [ "$v" = new ]; then lp=""; else lp="GM_LIB_PATH=$PWD/ab_libs/old/libgpumux_b200.so"; fi
  for m in mix resnet50; do
    for b in 4 8; do
      env $lp timeout 120 python tools/trace_round.py --model $m --tenants 4 --batch $b --out gpurun_out/abm_${v}_${m}_$b.json > gpurun_out/abm_${v}_${m}_$b.txt 2>&1 || echo fail
      echo "$v $m b$b: $(tail -1 gpurun_out/abm_${v}_${m}_$b.txt)"
    done
  done
done
