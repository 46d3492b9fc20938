# end-of-round re-check after the training-step changes: all GPU tests, smoke, the default bench
# line, the training-step launch list and one ncu full capture of the saved-tile layer backward
mkdir -p gpurun_out/final3
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final3/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final3/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final3/bench_products.json 2> gpurun_out/final3/bench_products.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/launches_train.csv env K=5 python tools/train_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer_bwd -s 3 -c 1 -o gpurun_out/final3/prof_layer_bwd_saved env K=3 python tools/train_probe.py > /dev/null 2>&1
echo done
