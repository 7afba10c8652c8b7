mkdir -p gpurun_out
set -x
python -m pytest tests/test_sliced_model.py tests/test_gpu_sliced.py -x -q -m gpu > gpurun_out/pytest16.log 2>&1; echo rc=$? >> gpurun_out/pytest16.log
python tools/breakdown_sliced.py 1024x1024x1024 32 > gpurun_out/bd16_1024.log 2>&1
python tools/breakdown_sliced.py 512x512x512 16 > gpurun_out/bd16_512.log 2>&1
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b16_c2.json 2> gpurun_out/b16_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1024_16.csv python tools/breakdown_sliced.py 1024x1024x1024 32 > gpurun_out/ncu16.log 2>&1
echo done
