# training-step launch list (products, one batch per step) and host/wall time per step
out=gpurun_out/${1:-train}
mkdir -p $out
K=20 timeout 600 python tools/train_probe.py > $out/train_probe.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_train.csv env K=5 python tools/train_probe.py > /dev/null 2>> $out/err.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sage_hidden_bwd -s 4 -c 2 -o $out/full_hidden_bwd env K=3 python tools/train_probe.py > /dev/null 2>> $out/err.txt
echo done
