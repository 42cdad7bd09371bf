# ncu --set full of one staged CUDA-core micro launch (tools/pool_micro.py case $1)
timeout 300 env REPS=2 ncu --set full --clock-control none --import-source on -k regex:superkernel -s 3 -c 1 \
  -o gpurun_out/prof_$1 -f python tools/pool_micro.py $1 > gpurun_out/ncu_$1.log 2>&1
tail -2 gpurun_out/ncu_$1.log
