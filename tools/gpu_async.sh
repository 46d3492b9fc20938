# cp.async ring form: parity + slot-count A/B against the pipelined default
CMB_AGG_KERNEL=a timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_async.log 2>&1
timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/as_pipe.json 2>>gpurun_out/as.err
for k in 8 12 16 24; do
  CMB_AGG_KERNEL=a CMB_ASYNC_SLOTS=$k timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/as_$k.json 2>>gpurun_out/as.err
done
timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/as_pipe2.json 2>>gpurun_out/as.err
echo done
