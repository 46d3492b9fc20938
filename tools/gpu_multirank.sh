# multi-rank bench flow on ONE GPU (2 ranks share cuda:0, gloo for the host collectives)
CMB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 40 --warmup 4 --no-extra --cpu-seconds 1 > gpurun_out/mr_cmb.json 2> gpurun_out/mr_cmb.err
echo "rc=$?" >> gpurun_out/mr_cmb.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "rc=$?" >> gpurun_out/mr_ref.err
echo done
