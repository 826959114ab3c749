# K1 over PEER (simulated ranks): row engine vs the bulk-copy pipeline (the
# default), W = 2/4/8, and the chunk count of the W = 8 ring; parity tests
# with the row engine forced.
echo rows; TW_K1_PEER_ENGINE=rows python tools/tp_colocated_sweep.py 2>&1 | grep '"tp": [248]'
echo tma; python tools/tp_colocated_sweep.py 2>&1 | grep '"tp": [248]'
echo tma-chunks3; TW_K1_PEER_CHUNKS=3 python tools/tp_colocated_sweep.py 2>&1 | grep '"tp": [48]'
TW_K1_PEER_ENGINE=rows timeout 900 python -m pytest tests/test_k1_gpu.py tests/test_soak_gpu.py -q -x -m gpu 2>&1 | tail -2
