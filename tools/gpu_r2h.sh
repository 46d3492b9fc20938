# round 2: sampler-written dst visiting order (cmb_blocks.dst_order) used by the fused gather
mkdir -p gpurun_out/r2h
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_peer.py tests/test_gpu_cache.py tests/test_gpu_papers.py -k "not papers_full" -x -q -p no:cacheprovider > gpurun_out/r2h/tests.log 2>&1
K=24 timeout 300 python tools/order_probe.py > gpurun_out/r2h/order.json 2>> gpurun_out/r2h/err.txt
NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2h/prof_nb4.json 2>> gpurun_out/r2h/err.txt
timeout 600 python bench.py --steps 400 --warmup 8 --no-extra > gpurun_out/r2h/bench.json 2>> gpurun_out/r2h/err.txt
K=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_gather_mean_row --csv --log-file gpurun_out/r2h/order_ncu.csv python tools/order_probe.py > /dev/null 2>> gpurun_out/r2h/err.txt
echo done
