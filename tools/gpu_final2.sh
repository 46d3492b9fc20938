# end-of-round measurement (papers100M lines kept from tools/gpu_final.sh's run: unchanged kernels)
mkdir -p gpurun_out/final2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final2/bench_products.json 2> gpurun_out/final2/bench_products.err
for c in tiny arxiv reddit; do
  timeout 900 python bench.py --config $c --steps 200 --cpu-seconds 5 > gpurun_out/final2/bench_$c.json 2> gpurun_out/final2/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches_products.csv python bench.py --steps 40 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/launches_train.csv env K=5 python tools/train_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_mean_row -s 5 -c 1 -o gpurun_out/final2/prof_row_products python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_hidden_bwd -s 2 -c 2 -o gpurun_out/final2/prof_hidden_bwd env K=3 python tools/train_probe.py > /dev/null 2>&1
echo done
