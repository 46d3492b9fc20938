# one bench line per BASELINE config that fits one GPU (products is the default line)
for c in tiny arxiv reddit; do
  timeout 900 python bench.py --config $c --steps 200 --cpu-seconds 5 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
echo done
