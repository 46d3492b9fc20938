timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests7.log 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/b7_$name.json 2>>gpurun_out/b7.err; }
run l32c4
run l16c2 CMB_AGG_LPR=16 CMB_AGG_CH=2
run l16c4 CMB_AGG_LPR=16 CMB_AGG_CH=4
run l8 CMB_AGG_LPR=8
run bulk CMB_AGG_KERNEL=bulk
echo done
