mkdir -p gpurun_out/r2k
for nb in 2 4; do NB=$nb timeout 300 python tools/nb_probe.py >> gpurun_out/r2k/nb.jsonl 2>> gpurun_out/r2k/err.txt; done
for nb in 4 6 8; do CMB_LIB_PATH=paper_2504_18082_b200/variants/libcmb_nb8.so NB=$nb timeout 300 python tools/nb_probe.py >> gpurun_out/r2k/nb.jsonl 2>> gpurun_out/r2k/err.txt; done
echo done
