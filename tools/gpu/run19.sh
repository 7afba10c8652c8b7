mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:update_rows -s 3 -c 1 -o gpurun_out/ncu19_update python tools/small_kernels.py 1024 32 > gpurun_out/ncu19a.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:normalize_gram -s 3 -c 1 -o gpurun_out/ncu19_norm python tools/small_kernels.py 1024 32 > gpurun_out/ncu19b.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bpp_kernel -s 3 -c 1 -o gpurun_out/ncu19_bpp python tools/small_kernels.py 1024 32 > gpurun_out/ncu19c.log 2>&1
echo done
