# round 2: dst-row visiting order probe (times + ncu DRAM bytes), GCN backward parity
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "gcn" > gpurun_out/r2c/tests_gcn.log 2>&1
for sh in 8 10 12; do SHIFT=$sh timeout 300 python tools/order_probe.py >> gpurun_out/r2c/order.jsonl 2>> gpurun_out/r2c/order.err; done
MODE=comm MIX=0.125 P=1.0 timeout 300 python tools/order_probe.py >> gpurun_out/r2c/order.jsonl 2>> gpurun_out/r2c/order.err
K=6 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_gather_mean_row --csv --log-file gpurun_out/r2c/order_ncu.csv python tools/order_probe.py > /dev/null 2>> gpurun_out/r2c/order.err
echo done
