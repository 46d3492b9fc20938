# A/B of library variants in one session: bench lines with CMB_LIB_PATH=<variant .so> (built with
# _build.build(out=..., defines=...) into gpurun_variants/, untracked) or "intree", two rounds,
# each variant with every bench flag set given in $3 (";"-separated, e.g. "--dst-order on;--dst-order off")
out=gpurun_out/${1:-vab}
libs=$2
IFS=';' read -ra modes <<< "${3:-}"
[ ${#modes[@]} -eq 0 ] && modes=("")
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_headline.py tests/test_gpu_peer.py -x -q -p no:cacheprovider > $out/tests.log 2>&1
for r in ${ROUNDS:-1 2}; do
  for v in $libs; do
    name=$(basename $v .so)
    if [ "$v" = "intree" ]; then lib=""; else lib=$v; fi
    for i in "${!modes[@]}"; do
      CMB_LIB_PATH=$lib timeout 600 python bench.py --steps 400 --warmup 8 --no-extra --cpu-seconds 0.5 ${modes[$i]} > $out/${name}_m${i}_$r.json 2>> $out/err.txt
    done
  done
done
echo done
