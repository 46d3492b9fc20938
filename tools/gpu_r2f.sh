mkdir -p gpurun_out/r2f
NB=4 timeout 300 python tools/profile_sampler.py > gpurun_out/r2f/prof_nb4.json 2>> gpurun_out/r2f/err.txt
NB=1 timeout 300 python tools/profile_sampler.py > gpurun_out/r2f/prof_nb1.json 2>> gpurun_out/r2f/err.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_persistent -s 3 -c 1 -o gpurun_out/r2f/sampler_full python bench.py --steps 16 --warmup 8 --no-extra --cpu-seconds 0.5 > /dev/null 2>> gpurun_out/r2f/err.txt
echo done
