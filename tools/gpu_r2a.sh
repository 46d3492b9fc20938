# round 2, first GPU session: the headline parity test + overlap A/B probes
mkdir -p gpurun_out/r2a
nproc > gpurun_out/r2a/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Socket|Thread" >> gpurun_out/r2a/host.txt; free -g >> gpurun_out/r2a/host.txt
( time timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -p no:cacheprovider ) > gpurun_out/r2a/headline.log 2>&1
for envs in "CMB_X=0" "CMB_SAMPLER_THREADS=512" "CMB_AGG_BLOCKS_PER_SM=2" "CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=2" "CMB_SAMPLER_THREADS=512 CMB_AGG_BLOCKS_PER_SM=3" "CMB_AGG_BLOCKS_PER_SM=3"; do
  env $envs timeout 300 python tools/overlap_probe.py >> gpurun_out/r2a/overlap.jsonl 2>>gpurun_out/r2a/overlap.err
done
echo done
