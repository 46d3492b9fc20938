timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "products_scaled or tiny or isolated" > gpurun_out/tests_mark.log 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 200 --no-extra --cpu-seconds 1 --mode comm --mix 0.0 --p 1.0 > gpurun_out/mk_${name}_m0.json 2>>gpurun_out/mk.err; env "$@" timeout 300 python bench.py --steps 200 --no-extra --cpu-seconds 1 > gpurun_out/mk_${name}_rand.json 2>>gpurun_out/mk.err; }
run check CMB_MARK_CHECK=1
run nocheck CMB_MARK_CHECK=0
run unfused_dedup CMB_FUSE_PICKS=0 CMB_PICK_DEDUP=1
run unfused CMB_FUSE_PICKS=0 CMB_PICK_DEDUP=0
echo done
