# round 2: full GPU suite after the knob cleanup + root range checks; bench multi-rank and
# sharded dry runs on one GPU; default bench line
mkdir -p gpurun_out/r2b
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/r2b/tests.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 8 > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
CMB_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 40 --warmup 4 --no-extra > gpurun_out/r2b/bench_gpus2_gloo.json 2> gpurun_out/r2b/bench_gpus2_gloo.err
timeout 600 python bench.py --shard a2a --steps 40 --warmup 4 > gpurun_out/r2b/bench_products_a2a.json 2> gpurun_out/r2b/bench_products_a2a.err
timeout 600 python bench.py --shard ipc --steps 40 --warmup 4 > gpurun_out/r2b/bench_products_ipc.json 2> gpurun_out/r2b/bench_products_ipc.err
CMB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config papers100m --shard ipc --steps 40 --warmup 4 > gpurun_out/r2b/bench_papers_ipc_gpus2.json 2> gpurun_out/r2b/bench_papers_ipc_gpus2.err
timeout 900 python bench.py --config papers100m --shard a2a --steps 40 --warmup 4 > gpurun_out/r2b/bench_papers_a2a.json 2> gpurun_out/r2b/bench_papers_a2a.err
echo done
