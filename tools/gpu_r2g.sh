# round 2: sampler with batched loads (counts RPT rows/thread, picks per row, flags/assign/relabel 8 edges/thread)
mkdir -p gpurun_out/r2g
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_batched.py tests/test_gpu_peer.py -x -q -p no:cacheprovider > gpurun_out/r2g/tests.log 2>&1
NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2g/prof_nb4.json 2>> gpurun_out/r2g/err.txt
NB=1 timeout 300 python tools/profile_sampler.py > gpurun_out/r2g/prof_nb1.json 2>> gpurun_out/r2g/err.txt
timeout 600 python bench.py --steps 200 --warmup 8 --no-extra > gpurun_out/r2g/bench.json 2>> gpurun_out/r2g/err.txt
echo done
