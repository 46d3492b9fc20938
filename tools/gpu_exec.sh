timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_exec.log 2>&1
timeout 600 python tools/host_probe.py > gpurun_out/host_probe2.json 2> gpurun_out/host_probe.err
timeout 600 python bench.py > gpurun_out/exec_products.json 2> gpurun_out/exec.err
echo done
