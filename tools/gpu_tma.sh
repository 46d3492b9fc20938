CMB_AGG_KERNEL=g timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q -p no:cacheprovider > gpurun_out/tests_tma.log 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/tma_$name.json 2>>gpurun_out/tma.err; }
run pipe CMB_AGG_KERNEL=p
run g4s2 CMB_AGG_KERNEL=g CMB_TMA_STAGES=2
run g4s3 CMB_AGG_KERNEL=g CMB_TMA_STAGES=3
run g4s4 CMB_AGG_KERNEL=g CMB_TMA_STAGES=4
run g4s2p0 CMB_AGG_KERNEL=g CMB_TMA_STAGES=2 CMB_TMA_L2PROMO=0
run g4s2p256 CMB_AGG_KERNEL=g CMB_TMA_STAGES=2 CMB_TMA_L2PROMO=256
echo done
