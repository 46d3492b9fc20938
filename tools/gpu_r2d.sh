# round 2: fused gather codegen A/B (predicated loads, uint32 row stride; MINB 4/3/2; dense vs
# one-shard ShardedRows), times in the probe and cold-L2 ncu counters
mkdir -p gpurun_out/r2d
for v in default minb3 minb2; do
  if [ $v = default ]; then lp=""; else lp="CMB_LIB_PATH=paper_2504_18082_b200/variants/libcmb_$v.so"; fi
  env $lp K=24 timeout 300 python tools/order_probe.py > gpurun_out/r2d/order_$v.json 2>> gpurun_out/r2d/err.txt
done
K=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_mean_row -s 0 -c 5 -o gpurun_out/r2d/gather_full python tools/order_probe.py > /dev/null 2>> gpurun_out/r2d/err.txt
timeout 600 python bench.py --steps 200 --warmup 8 --no-extra > gpurun_out/r2d/bench.json 2>> gpurun_out/r2d/err.txt
echo done
