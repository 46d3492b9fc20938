# compute-sanitizer evidence for the round-2 code paths (run on the box from the repo root)
out=gpurun_out/${1:-san}
mkdir -p $out
cs=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $cs --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $out/memcheck_smoke.txt 2>&1; echo "rc=$?" >> $out/memcheck_smoke.txt
timeout 1200 $cs --tool memcheck python bench.py --steps 8 --warmup 4 --no-extra --cpu-seconds 0.5 > $out/memcheck_bench.txt 2>&1; echo "rc=$?" >> $out/memcheck_bench.txt
timeout 1200 $cs --tool racecheck python -m pytest tests/test_gpu_batched.py -q -p no:cacheprovider -k "dst_order or multi" > $out/racecheck_sampler_order.txt 2>&1; echo "rc=$?" >> $out/racecheck_sampler_order.txt
timeout 1200 $cs --tool memcheck python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "dense or gcn_layer_backward" > $out/memcheck_dense_gcn.txt 2>&1; echo "rc=$?" >> $out/memcheck_dense_gcn.txt
timeout 1200 $cs --tool memcheck python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "isolated or ragged or bad_input or capacity or out_of_range or row_offsets" > $out/memcheck_edge.txt 2>&1; echo "rc=$?" >> $out/memcheck_edge.txt
timeout 1500 $cs --tool memcheck python -m pytest tests/test_gpu_mapword.py -q -p no:cacheprovider > $out/memcheck_mapword.txt 2>&1; echo "rc=$?" >> $out/memcheck_mapword.txt
timeout 1200 $cs --tool synccheck python -m pytest tests/test_gpu_batched.py -q -p no:cacheprovider -k "multi" > $out/synccheck_sampler.txt 2>&1; echo "rc=$?" >> $out/synccheck_sampler.txt
echo done
