# A/B runs on the GPU box (called through gpurun); every leg under its own timeout.
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests8.log 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/b8_$name.json 2>>gpurun_out/b8.err; }
run persist
run multi CMB_SAMPLER=multi
echo done
