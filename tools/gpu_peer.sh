timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_peer.log 2>&1
timeout 600 python tools/peer_timing.py > gpurun_out/peer_timing.json 2> gpurun_out/peer_timing.err
echo done
