# A/B runs on the GPU box: run `bash tools/gpu_ab.sh TAG name1 "ENV=.." name2 "ENV=.." ...`
tag=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_$tag.log 2>&1
while [ $# -gt 1 ]; do
  name=$1; envs=$2; shift 2
  env $envs timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/ab_${tag}_$name.json 2>>gpurun_out/ab_$tag.err
done
echo done
