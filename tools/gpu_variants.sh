# A/B of layout variants (libraries built by _build.build(out=..., defines=...) under
# paper_2504_18082_b200/variants/): whole-step us per batch at 4 batches per launch, twice each
mkdir -p gpurun_out/variants
rm -f gpurun_out/variants/nb.jsonl
for r in 1 2; do
  echo "{\"variant\": \"default\"}" >> gpurun_out/variants/nb.jsonl
  NB=4 timeout 300 python tools/nb_probe.py >> gpurun_out/variants/nb.jsonl 2>> gpurun_out/variants/err.txt
  for v in $(ls paper_2504_18082_b200/variants/ | sed 's/libcmb_//; s/.so//'); do
    echo "{\"variant\": \"$v\"}" >> gpurun_out/variants/nb.jsonl
    CMB_LIB_PATH=paper_2504_18082_b200/variants/libcmb_$v.so NB=4 timeout 300 python tools/nb_probe.py >> gpurun_out/variants/nb.jsonl 2>> gpurun_out/variants/err.txt
  done
done
echo done
