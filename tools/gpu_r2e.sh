# round 2: unconditional-load form of the fused gather: parity + times + ncu
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_peer.py tests/test_gpu_cache.py tests/test_gpu_batched.py -x -q -p no:cacheprovider > gpurun_out/r2e/tests.log 2>&1
K=24 timeout 300 python tools/order_probe.py > gpurun_out/r2e/order.json 2>> gpurun_out/r2e/err.txt
timeout 600 python bench.py --steps 200 --warmup 8 --no-extra > gpurun_out/r2e/bench.json 2>> gpurun_out/r2e/err.txt
timeout 600 python bench.py --config reddit --steps 100 --warmup 8 --no-extra > gpurun_out/r2e/bench_reddit.json 2>> gpurun_out/r2e/err.txt
K=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_mean_row -s 0 -c 5 -o gpurun_out/r2e/gather_full python tools/order_probe.py > /dev/null 2>> gpurun_out/r2e/err.txt
echo done
