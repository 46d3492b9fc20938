mkdir -p gpurun_out/pp
CFG=papers100m K=12 timeout 900 python tools/order_probe.py > gpurun_out/pp/order_papers.json 2> gpurun_out/pp/err.txt
K=12 timeout 300 python tools/order_probe.py > gpurun_out/pp/order_products.json 2>> gpurun_out/pp/err.txt
echo done
