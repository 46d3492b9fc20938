mkdir -p gpurun_out/tl
NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/tl/nb4.json 2> gpurun_out/tl/err.txt
echo done
