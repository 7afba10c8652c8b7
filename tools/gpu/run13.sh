mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,power.limit,power.max_limit,clocks.max.sm,clocks.max.mem,temperature.gpu --format=csv > gpurun_out/smi13.txt 2>&1
python tools/breakdown_sliced.py 2048x2048x2048 32 > gpurun_out/bd13.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b13_c5.json 2> gpurun_out/b13_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_13.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu13.log 2>&1
echo done
