# hot-path change check: sampler + gather parity (incl. the headline path), two short bench
# lines, the sampler timeline and ncu --set full of the gather and the sampler
out=gpurun_out/${1:-pc}
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_mapword.py tests/test_gpu_batched.py tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q -p no:cacheprovider > $out/tests.log 2>&1
for r in 1 2; do timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 > $out/bench_$r.json 2>> $out/err.txt; done
NB=6 timeout 300 python tools/profile_sampler.py > $out/timeline.json 2>> $out/err.txt
for k in k_gather_mean_row k_sample_persistent; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 8 -c 1 \
    -o $out/full_$k python bench.py --steps 16 --warmup 8 --no-extra --cpu-seconds 1 > /dev/null 2>> $out/ncu.err
done
echo done
