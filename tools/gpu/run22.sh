mkdir -p gpurun_out
set -x
for c in c2 c5blk8 c3; do
  NNCP_PDL=0 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b22_${c}_off.json 2> gpurun_out/b22_${c}_off.err
  NNCP_PDL=1 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b22_${c}_wait.json 2> gpurun_out/b22_${c}_wait.err
  NNCP_LIB_PATH=$PWD/paper_1909_01149_b200/libnncp_b200_early.so NNCP_PDL=1 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b22_${c}_early.json 2> gpurun_out/b22_${c}_early.err
  NNCP_PDL=0 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b22_${c}_off2.json 2> gpurun_out/b22_${c}_off2.err
done
echo done
