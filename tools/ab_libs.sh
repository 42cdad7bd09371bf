# A/B of library variants (ab_libs/<name>/libgpumux_b200.so, GM_LIB_PATH) on the headline round trace
for v in default ${VARIANTS}; do
  if [ "$v" = default ]; then lp=""; else lp="GM_LIB_PATH=$PWD/ab_libs/$v/libgpumux_b200.so"; fi
  for rep in 1 2; do
    env $lp timeout 120 python tools/trace_round.py --out gpurun_out/ab_$v.json > gpurun_out/ab_$v.txt 2>&1 || echo "$v failed: $(tail -2 gpurun_out/ab_$v.txt)"
    echo "$v: $(tail -1 gpurun_out/ab_$v.txt)"
  done
done
