mkdir -p gpurun_out/rr
timeout 1500 python -m pytest tests/test_gpu_reorder.py tests/test_gpu_papers.py tests/test_gpu_batched.py -q -p no:cacheprovider > gpurun_out/rr/tests.log 2>&1
echo done
