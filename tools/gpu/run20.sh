mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"bseg_|ttv_leading" -s 6 -c 3 -o gpurun_out/ncu20_prep python bench.py --config c5blk8 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu20.log 2>&1
echo done
