set -x
o=gpurun_out/m3
mkdir -p $o
./build/bench/dropin_bench phases 8192 8192 3 > $o/phases.json 2>&1
./build/bench/dropin_bench rmsnorm 8192 8192 2 5 > $o/dropin.json 2>&1
timeout 1200 python -m pytest tests/test_k1_gpu.py tests/test_nvls_gpu.py tests/test_soak_gpu.py tests/test_mp_gpu.py -m gpu -q -x -p no:cacheprovider > $o/tests.txt 2>&1
tail -3 $o/tests.txt
timeout 300 python tools/k1_small.py > $o/k1_small_dev.txt 2>&1
TW_FORCE_SYS_SCOPE=1 timeout 300 python tools/k1_small.py > $o/k1_small_sys.txt 2>&1
timeout 300 python tools/k1_small.py --transport nvls_sim > $o/k1_small_nvlssim.txt 2>&1
echo done
