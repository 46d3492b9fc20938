# sampler change check: sampler parity tests (incl. the headline path) + two short bench lines
out=gpurun_out/${1:-sc}
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_mapword.py tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q -p no:cacheprovider > $out/tests.log 2>&1
for r in 1 2; do timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 > $out/bench_$r.json 2>> $out/err.txt; done
NB=6 timeout 300 python tools/profile_sampler.py > $out/timeline.json 2>> $out/err.txt
echo done
