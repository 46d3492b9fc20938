# NEXT-4 measurement: bench layer point on products + arxiv, ncu full capture of k_sage_layer
mkdir -p gpurun_out/layer
timeout 600 python bench.py --steps 50 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/bench_products.json 2> gpurun_out/layer/bench_products.err
timeout 600 python bench.py --config arxiv --steps 50 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/bench_arxiv.json 2> gpurun_out/layer/bench_arxiv.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer -s 5 -c 1 -o gpurun_out/layer/prof_layer_products python bench.py --steps 4 --warmup 3 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/ncu.log 2>&1
echo done
