mkdir -p gpurun_out
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest21.log 2>&1; echo rc=$? >> gpurun_out/pytest21.log
for c in c2 c5blk8 c3 c5; do
  for pdl in 1 0; do
    NNCP_PDL=$pdl python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b21_${c}_pdl$pdl.json 2> gpurun_out/b21_${c}_pdl$pdl.err
  done
done
echo done
