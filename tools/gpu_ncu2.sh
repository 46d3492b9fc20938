CMB_AGG_KERNEL=a CMB_ASYNC_SLOTS=8 timeout 600 ncu --set full --import-source on -k regex:k_gather_mean_async -s 5 -c 1 -o gpurun_out/prof_async8 python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_gather_mean_pipe -s 5 -c 1 -o gpurun_out/prof_pipe_fm python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 >> gpurun_out/ncu2.log 2>&1
echo done
