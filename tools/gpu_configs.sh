# Bench lines of every BASELINE.json config on one B200 (run from the repo root on the box):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_configs.sh r02'
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
for c in tiny arxiv reddit; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 8 --layer --cpu-seconds 6 \
    > $out/bench_$c.json 2> $out/bench_$c.err
done
timeout 1500 python bench.py --config papers100m --steps 200 --warmup 8 --no-extra --cpu-seconds 6 \
  > $out/bench_papers100m.json 2> $out/bench_papers100m.err
echo done
