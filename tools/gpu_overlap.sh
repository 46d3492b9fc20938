run() { name=$1; shift; env "$@" timeout 300 python tools/overlap_probe.py > gpurun_out/ov_$name.json 2>>gpurun_out/ov.err; }
run default
run s512_g1 CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=1
run s512_g2 CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=2
run s1024_g1 CMB_AGG_BLOCKS_PER_SM=1
run multi_g2 CMB_SAMPLER=multi CMB_AGG_BLOCKS_PER_SM=2
run multi CMB_SAMPLER=multi
echo done
