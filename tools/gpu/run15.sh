mkdir -p gpurun_out
set -x
(cd abtest/old && python bench.py --steps 10 --warmup 3 --no-cpu-baseline) > gpurun_out/b15_old1.json 2> gpurun_out/b15_old1.err
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b15_new1.json 2> gpurun_out/b15_new1.err
(cd abtest/old && python bench.py --steps 10 --warmup 3 --no-cpu-baseline) > gpurun_out/b15_old2.json 2> gpurun_out/b15_old2.err
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b15_new2.json 2> gpurun_out/b15_new2.err
echo done
