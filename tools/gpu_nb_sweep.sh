mkdir -p gpurun_out/nbsweep
for nb in 1 2 3 4; do NB=$nb timeout 300 python tools/nb_probe.py >> gpurun_out/nbsweep/nb.jsonl 2>> gpurun_out/nbsweep/err.txt; done
echo done
