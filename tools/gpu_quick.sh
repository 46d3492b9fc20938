# quick check of the path: parity of the sampler / gather entry points + two default bench lines
# + the sampler's per-phase timeline
mkdir -p gpurun_out/q
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_batched.py tests/test_gpu_peer.py tests/test_gpu_cache.py -x -q -p no:cacheprovider > gpurun_out/q/tests.log 2>&1
for r in 1 2; do timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 > gpurun_out/q/bench_$r.json 2>> gpurun_out/q/err.txt; done
NB=6 timeout 300 python tools/profile_sampler.py > gpurun_out/q/timeline.json 2>> gpurun_out/q/err.txt
echo done
