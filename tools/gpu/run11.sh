mkdir -p gpurun_out
set -x
python -m pytest tests/test_sliced_model.py tests/test_gpu_sliced.py -x -q -m gpu > gpurun_out/pytest11.log 2>&1; echo rc=$? >> gpurun_out/pytest11.log
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b11_c4.json 2> gpurun_out/b11_c4.err
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b11_c5.json 2> gpurun_out/b11_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c4_11.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu11.log 2>&1
echo done
