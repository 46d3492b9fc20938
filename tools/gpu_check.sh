# one GPU check of the current tree: the whole -m gpu suite, smoke() and the default bench line
mkdir -p gpurun_out/chk
( time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ) > gpurun_out/chk/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err
echo done
