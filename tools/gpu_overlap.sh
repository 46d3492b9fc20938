run() { name=$1; shift; env "$@" timeout 300 python tools/overlap_probe.py > gpurun_out/ov_$name.json 2>>gpurun_out/ov.err; }
run default
run s512_g2 CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=2
run s1024_g2 CMB_AGG_BLOCKS_PER_SM=2
run s512_g3 CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=3
echo done
