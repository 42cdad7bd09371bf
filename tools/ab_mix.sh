# Same-box A/B of the working-tree library ("new") against ab_libs/old on the
# headline, mix and BERT round traces (alternating, twice each)
set +e
for v in new old new old; do
  if [ "$v" = new ]; then lp=""; else lp="GM_LIB_PATH=$PWD/ab_libs/old/libgpumux_b200.so"; fi
  for mb in resnet50:4:8 mix:4:4 bert:16:4; do
    m=${mb%%:*}; t=$(echo $mb | cut -d: -f2); b=${mb##*:}
    env $lp timeout 120 python tools/trace_round.py --model $m --tenants $t --batch $b --out gpurun_out/abm_${v}_${m}.json > gpurun_out/abm_${v}_${m}.txt 2>&1 || echo fail
    echo "$v $m b$b: $(tail -1 gpurun_out/abm_${v}_${m}.txt)"
  done
done
