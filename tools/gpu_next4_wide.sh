mkdir -p gpurun_out/r2l
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_train.py -q -p no:cacheprovider -x > gpurun_out/r2l/tests.log 2>&1
timeout 900 python bench.py --config reddit --steps 100 --warmup 8 --no-extra --layer --cpu-seconds 2 > gpurun_out/r2l/bench_reddit.json 2> gpurun_out/r2l/bench_reddit.err
echo done
