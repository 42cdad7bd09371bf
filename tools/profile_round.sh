# Round-end profiling recipe (B200_PROFILING.md): bench line, launch list, one
# ncu --set full capture of the round-program super-kernel.  Writes gpurun_out/.
set -x
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --table1 '' --cpu-seconds 0.1 --serve-seconds 0 --extra '' > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:superkernel -s 1 -c 1 \
  -o gpurun_out/prof_round -f python tools/ncu_target.py --round --rounds 2 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
