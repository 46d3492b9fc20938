# batches-per-launch sweep (tools/nb_probe.py) for library variants built with a larger
# CMB_MAX_BATCHES_PER_LAUNCH, at RAND p = 0.5 and at the contended knob points (MIX-0 / NORAND, p = 1)
out=gpurun_out/${1:-nbs}
shift
mkdir -p $out
for r in 1 2; do
  for lib in "$@"; do
    name=$(basename $lib .so)
    for nb in 4 5 6 7 8; do NB=$nb CMB_LIB_PATH=$lib timeout 300 python tools/nb_probe.py > $out/${name}_rand_nb${nb}_$r.json 2>> $out/err.txt; done
    for nb in 4 6; do
      NB=$nb MODE=comm MIX=0 P=1.0 CMB_LIB_PATH=$lib timeout 300 python tools/nb_probe.py > $out/${name}_mix0_nb${nb}_$r.json 2>> $out/err.txt
      NB=$nb MODE=norand P=1.0 CMB_LIB_PATH=$lib timeout 300 python tools/nb_probe.py > $out/${name}_norand_nb${nb}_$r.json 2>> $out/err.txt
    done
  done
done
echo done
