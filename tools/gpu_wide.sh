timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "reddit or products_scaled or isolated" > gpurun_out/tests_wide.log 2>&1
for d in 4 5 6 8; do
CMB_ROW_DMAX=$d timeout 900 python bench.py --config reddit --steps 200 --cpu-seconds 1 --no-extra > gpurun_out/wide_reddit$d.json 2>> gpurun_out/wide.err
done
timeout 900 python bench.py --steps 300 --cpu-seconds 1 --no-extra > gpurun_out/wide_products.json 2>> gpurun_out/wide.err
echo done
