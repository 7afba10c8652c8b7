mkdir -p gpurun_out
set -x
python tools/small_kernels.py 2048 32 > gpurun_out/sk17_2048.log 2>&1
python tools/small_kernels.py 1024 32 > gpurun_out/sk17_1024.log 2>&1
python tools/small_kernels.py 512 16 > gpurun_out/sk17_512.log 2>&1
python bench.py --config c5blk8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b17_blk8.json 2> gpurun_out/b17_blk8.err
echo done
