mkdir -p gpurun_out/knobs
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for c in products arxiv reddit; do
  CFG=$c timeout 900 python tools/knob_counters.py > gpurun_out/knobs/$c.plain.jsonl 2> gpurun_out/knobs/$c.err
  CFG=$c timeout 1200 ncu --metrics $M --clock-control none -k regex:k_gather_mean_row --csv --log-file gpurun_out/knobs/$c.ncu.csv python tools/knob_counters.py > gpurun_out/knobs/$c.ncu.jsonl 2>> gpurun_out/knobs/$c.err
  python tools/knob_counters_summary.py gpurun_out/knobs/$c.plain.jsonl gpurun_out/knobs/$c.ncu.csv > gpurun_out/knobs/$c.summary.json 2>> gpurun_out/knobs/$c.err
done
echo done
