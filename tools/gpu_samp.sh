timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "products or tiny or ragged" > gpurun_out/tests_samp.log 2>&1
for cfg in "h1d1 CMB_STREAM_HINT=1 CMB_PICK_DEDUP=1" "h0d1 CMB_STREAM_HINT=0 CMB_PICK_DEDUP=1" "h1d0 CMB_STREAM_HINT=1 CMB_PICK_DEDUP=0" "h0d0 CMB_STREAM_HINT=0 CMB_PICK_DEDUP=0" "h1d1b CMB_STREAM_HINT=1 CMB_PICK_DEDUP=1"; do
  set -- $cfg; name=$1; shift
  env "$@" timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/sh_$name.json 2>>gpurun_out/sh.err
done
echo done
