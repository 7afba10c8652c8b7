mkdir -p gpurun_out
set -x
python tools/small_kernels.py 1024 32 > gpurun_out/sk18_1024.log 2>&1
python tools/small_kernels.py 2048 32 > gpurun_out/sk18_2048.log 2>&1
python tools/small_kernels.py 512 16 > gpurun_out/sk18_512.log 2>&1
python tools/small_kernels.py 256 32 > gpurun_out/sk18_256.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest18.log 2>&1; echo rc=$? >> gpurun_out/pytest18.log
python bench.py --config c5blk8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b18_blk8.json 2> gpurun_out/b18_blk8.err
python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b18_c2.json 2> gpurun_out/b18_c2.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b18_c3.json 2> gpurun_out/b18_c3.err
echo done
