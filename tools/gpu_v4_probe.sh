out=gpurun_out/vab4
mkdir -p $out
for r in 1 2; do
  for v in intree gpurun_variants/libcmb_noprecheck.so; do
    name=$(basename $v .so); lib=""; [ "$v" != "intree" ] && lib=$v
    CMB_LIB_PATH=$lib timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 > $out/${name}_$r.json 2>> $out/err.txt
  done
  for nb in 4 6 8; do NB=$nb CMB_LIB_PATH=gpurun_variants/libcmb_nb8.so timeout 300 python tools/nb_probe.py > $out/nb${nb}_$r.json 2>> $out/err.txt; done
done
echo done
