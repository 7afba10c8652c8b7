mkdir -p gpurun_out
set -x
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b12_c5a.json 2> gpurun_out/b12_c5a.err
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b12_c2.json 2> gpurun_out/b12_c2.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b12_c3.json 2> gpurun_out/b12_c3.err
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b12_c5b.json 2> gpurun_out/b12_c5b.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_12.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu12a.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3_12.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu12b.log 2>&1
echo done
