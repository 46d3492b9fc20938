# measurement round: tests, smoke, every config's bench line, launch list + ncu captures
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_products.json 2> gpurun_out/final/bench_products.err
for c in tiny arxiv reddit; do
  timeout 900 python bench.py --config $c --steps 200 --cpu-seconds 5 > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_products.csv python bench.py --steps 40 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_mean_row -s 5 -c 1 -o gpurun_out/final/prof_row_products python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_persistent -s 3 -c 1 -o gpurun_out/final/prof_sampler_products python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 1800 python bench.py --config papers100m --steps 200 --cpu-seconds 20 > gpurun_out/final/bench_papers100m.json 2> gpurun_out/final/bench_papers100m.err
timeout 900 ncu --set full --clock-control none -k regex:k_gather_mean_row -s 5 -c 1 -o gpurun_out/final/prof_row_papers python bench.py --config papers100m --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1

timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer -s 8 -c 2 -o gpurun_out/final/prof_layer_products python bench.py --steps 4 --warmup 3 --no-extra --layer --cpu-seconds 1 > /dev/null 2>&1
echo done2
