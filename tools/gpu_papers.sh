# papers100M-shaped: scaled + full parity, then the single-GPU bench line (graph replicated)
timeout 600 python -m pytest tests/test_gpu_papers.py -m gpu -x -q -p no:cacheprovider -k scaled > gpurun_out/tests_papers_scaled.log 2>&1
( time CMB_TEST_PAPERS=1 timeout 2400 python -m pytest tests/test_gpu_papers.py -m gpu -x -q -s -p no:cacheprovider -k full ) > gpurun_out/tests_papers_full.log 2>&1
free -g >> gpurun_out/tests_papers_full.log
timeout 1800 python bench.py --config papers100m --steps 200 --cpu-seconds 20 > gpurun_out/bench_papers.json 2> gpurun_out/bench_papers.err
echo done
