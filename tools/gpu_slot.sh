timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_slot.log 2>&1
timeout 300 python bench.py --steps 300 --no-extra --cpu-seconds 1 > gpurun_out/slot_a.json 2> gpurun_out/slot.err
echo done
