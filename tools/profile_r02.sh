# Profiling pass (B200_PROFILING.md recipe): launch list of the bench command,
# one ncu --set full capture of the round-program kernel per config, and an
# in-kernel trace of the headline round.  Writes gpurun_out/.
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --table1 '' --cpu-seconds 0.1 --serve-seconds 0 --extra '' > gpurun_out/ncu_bench.log 2>&1
for c in ${CONFIGS:-headline bert4 mix4 table1}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:superkernel -s 1 -c 1 \
    -o gpurun_out/prof_$c -f python tools/ncu_target.py --config $c --round --rounds 2 > gpurun_out/ncu_$c.log 2>&1
done
timeout 120 python tools/trace_round.py --out gpurun_out/tr_default.json > gpurun_out/tr_default.txt 2>&1
ls -la gpurun_out
