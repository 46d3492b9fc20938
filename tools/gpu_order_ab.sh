# bench A/B of the sampler-written dst visiting order (same bytes either way)
mkdir -p gpurun_out/order_ab
for r in 1 2; do
  for o in off on; do
    timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 --dst-order $o > gpurun_out/order_ab/products_${o}_$r.json 2>> gpurun_out/order_ab/err.txt
  done
done
for o in off on; do
  timeout 1500 python bench.py --config papers100m --steps 200 --warmup 8 --no-extra --cpu-seconds 0.5 --dst-order $o > gpurun_out/order_ab/papers_${o}.json 2>> gpurun_out/order_ab/err.txt
done
echo done
