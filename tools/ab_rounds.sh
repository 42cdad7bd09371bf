# Same-box A/B of round programs (debug aid): AB_LIBS="base cur" AB_CONFIGS="headline mix bert4" AB_OPTS="-"
for rep in 1 2; do for c in ${AB_CONFIGS:-headline}; do for lib in ${AB_LIBS:-base cur}; do
  if [ "$lib" = cur ]; then L=""; else L=paper_1901_00041_b200/_lib/$lib/libgpumux_b200.so; fi
  echo -n "$lib "; GM_LIB_PATH=$L timeout 300 python tools/round_ab.py --config $c --reps 1 --opts ${AB_OPTS:--}
done; done; done
