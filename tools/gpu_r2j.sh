mkdir -p gpurun_out/r2j
for v in store cheaprng; do
  CMB_LIB_PATH=paper_2504_18082_b200/variants/libcmb_cmb_exp_$v.so NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2j/prof_$v.json 2>> gpurun_out/r2j/err.txt
done
echo done
