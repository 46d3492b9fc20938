for cfg in "d6m4 CMB_ROW_DMAX=6" "d5m4 CMB_ROW_DMAX=5" "d5m5 CMB_ROW_DMAX=5 CMB_ROW_MINB=5" "d6m5 CMB_ROW_DMAX=6 CMB_ROW_MINB=5" "d4m5 CMB_ROW_DMAX=4 CMB_ROW_MINB=5" "d6m4b4 CMB_ROW_DMAX=6 CMB_AGG_BLOCKS_PER_SM=4" "d6m4b16 CMB_ROW_DMAX=6 CMB_AGG_BLOCKS_PER_SM=16" "d6m4r CMB_ROW_DMAX=6"; do
  set -- $cfg; name=$1; shift
  env CMB_AGG_KERNEL=w "$@" timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/rw_$name.json 2>>gpurun_out/rw.err
done
echo done
