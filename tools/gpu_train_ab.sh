# A/B of library variants on the NEXT-4 training point (bench --layer): layer / backward times and
# training steps per second, two rounds each; the layer / training parity tests on the in-tree lib
out=gpurun_out/${1:-tab}
libs=$2
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_train.py -q -x -p no:cacheprovider > $out/tests.log 2>&1
for r in 1 2; do for v in $libs; do
  name=$(basename $v .so); lib=""; [ "$v" != "intree" ] && lib=$v
  CMB_LIB_PATH=$lib timeout 900 python bench.py --no-extra --layer --steps 50 --warmup 8 --cpu-seconds 0.5 > $out/${name}_$r.json 2>> $out/err.txt
done; done
echo done
