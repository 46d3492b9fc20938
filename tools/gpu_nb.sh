timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_nb.log 2>&1
for nb in 4 6 8 4; do
  timeout 300 python bench.py --steps 400 --no-extra --cpu-seconds 1 --batches-per-launch $nb > gpurun_out/nb_$nb.json 2>>gpurun_out/nb.err
done
echo done
