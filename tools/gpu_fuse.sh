timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_fuse.log 2>&1
CMB_FUSE_PICKS=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "products_scaled or slot" > gpurun_out/tests_fuse0.log 2>&1
for f in 1 0 1 0; do
  CMB_FUSE_PICKS=$f timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/fu_$f.json 2>> gpurun_out/fu.err
done
NB=4 timeout 600 python tools/profile_sampler.py > gpurun_out/psf_4.json 2>> gpurun_out/fu.err
echo done
