mkdir -p gpurun_out/layer
timeout 600 python bench.py --steps 20 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/bench_products.json 2>/dev/null
timeout 600 python bench.py --config arxiv --steps 20 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/bench_arxiv.json 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer -s 8 -c 2 -o gpurun_out/layer/prof_layer_v3 python bench.py --steps 4 --warmup 3 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/ncu.log 2>&1
echo done
