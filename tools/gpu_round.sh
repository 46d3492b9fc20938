# full GPU round: tests, smoke, default bench, launch list + ncu full capture of the gather kernel
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_round.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_round.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_round.csv python bench.py --steps 40 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_mean_row -s 5 -c 1 -o gpurun_out/prof_row python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 > gpurun_out/ncu_row.log 2>&1
echo done
