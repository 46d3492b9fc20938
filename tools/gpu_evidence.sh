# The round's GPU evidence in one gpurun call (run from the repo root on the B200 box):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_evidence.sh r02'
# -> gpurun_out/<tag>/: the -m gpu suite, smoke(), the default bench line, the ncu launch list
# of that same bench command (cold, serialised), one ncu --set full capture of each top kernel
# (fused gather, sampler, fused layer 1), the DRAM counters per knob point, and the sampler's
# per-phase timeline.  tools/ncu_*_summary.py turn the .ncu-rep / csv files into profiles/.
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nproc > $out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $out/host.txt
( time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $out/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 16 --warmup 8 --no-extra --cpu-seconds 1 \
  > /dev/null 2>> $out/ncu.err
for k in k_gather_mean_row k_sample_persistent; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 8 -c 1 \
    -o $out/full_$k python bench.py --steps 16 --warmup 8 --no-extra --cpu-seconds 1 \
    > /dev/null 2>> $out/ncu.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sage_layer -s 4 -c 1 \
  -o $out/full_k_sage_layer python bench.py --steps 8 --warmup 4 --no-extra --layer \
  --cpu-seconds 1 > /dev/null 2>> $out/ncu.err
NB=6 timeout 300 python tools/profile_sampler.py > $out/sampler_timeline.json 2>> $out/ncu.err
echo done
