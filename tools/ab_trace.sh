# Same-box A/B of round-program spans (debug aid): ABN="lib:opts ..." where lib is
# "cur" or a directory name under paper_1901_00041_b200/_lib/ holding another build.
# e.g. ABN="old:- cur:- cur:split_k=1" bash tools/ab_trace.sh
for rep in 1 2; do
for spec in $ABN; do
  lib=${spec%%:*}; o=${spec#*:}
  if [ "$lib" = cur ]; then L=""; else L=paper_1901_00041_b200/_lib/$lib/libgpumux_b200.so; fi
  if [ "$o" = "-" ]; then args=""; else args=$(echo $o | sed 's/,/ --opt /g; s/^/--opt /'); fi
  GM_LIB_PATH=$L timeout 120 python tools/trace_round.py $args --out gpurun_out/ab_${lib}_${o}_$rep.json > gpurun_out/ab_${lib}_${o}_$rep.txt 2>&1
  echo "$rep $lib $o: $(tail -1 gpurun_out/ab_${lib}_${o}_$rep.txt)"
done; done
