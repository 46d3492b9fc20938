# quick verification: gpu tests, smoke, default bench line
mkdir -p gpurun_out/check
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/check/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/check/bench_products.json 2> gpurun_out/check/bench_products.err
echo done
