mkdir -p gpurun_out/layer
timeout 600 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider > gpurun_out/layer/tests.log 2>&1
for f in 0 2 1; do
CMB_LAYER_KERNEL=$f timeout 600 python bench.py --steps 20 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/ab_products_$f.json 2>/dev/null
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer -s 5 -c 1 -o gpurun_out/layer/prof_layer_v2 python bench.py --steps 4 --warmup 3 --no-extra --layer --cpu-seconds 1 > gpurun_out/layer/ncu.log 2>&1
echo done
