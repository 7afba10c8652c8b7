mkdir -p gpurun_out
set -x
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b14_c5a.json 2> gpurun_out/b14_c5a.err
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b14_c5b.json 2> gpurun_out/b14_c5b.err
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b14_c4.json 2> gpurun_out/b14_c4.err
echo done
