# round 2: what bounds the sampler's positions step? timeline with picks' CSR loads / marks removed
mkdir -p gpurun_out/r2i
NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2i/prof_default.json 2>> gpurun_out/r2i/err.txt
for v in noload noatom nocheck; do
  CMB_LIB_PATH=paper_2504_18082_b200/variants/libcmb_cmb_exp_$v.so NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2i/prof_$v.json 2>> gpurun_out/r2i/err.txt
done
echo done
