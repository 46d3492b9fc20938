# §8.1: per knob point, plain timing + ncu DRAM / L2 counters of the fused gather (cold L2)
out=gpurun_out/${1:-knobs}
mkdir -p $out
for c in products arxiv reddit; do
  CFG=$c timeout 900 python tools/knob_counters.py > $out/plain_$c.jsonl 2>> $out/err.txt
  CFG=$c timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_gather_mean_row --csv --log-file $out/ncu_$c.csv python tools/knob_counters.py > /dev/null 2>> $out/err.txt
  python tools/knob_counters_summary.py $out/plain_$c.jsonl $out/ncu_$c.csv > $out/summary_$c.json 2>> $out/err.txt
done
echo done
