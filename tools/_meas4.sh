set -x
o=gpurun_out/m4
mkdir -p $o
./build/bench/dropin_bench phases 8192 8192 3 > $o/phases.json 2>&1
./build/bench/dropin_bench rmsnorm 8192 8192 2 5 > $o/dropin.json 2>&1
timeout 200 python bench.py --impl reference --steps 5 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err
timeout 1200 python -m pytest tests/test_k1_gpu.py tests/test_nvls_gpu.py tests/test_soak_gpu.py tests/test_mp_gpu.py tests/test_dropin.py -m gpu -q -x -p no:cacheprovider > $o/tests.txt 2>&1
tail -3 $o/tests.txt
timeout 300 python tools/k1_small.py > $o/k1_small_dev.txt 2>&1
TW_FORCE_SYS_SCOPE=1 timeout 300 python tools/k1_small.py > $o/k1_small_sys.txt 2>&1
timeout 300 python tools/k1_small.py --transport nvls_sim > $o/k1_small_nvlssim.txt 2>&1
TW_NVLS_ALIAS_FENCE=1 timeout 300 python tools/k1_small.py --transport nvls_sim > $o/k1_small_nvlssim_alias.txt 2>&1
for ring in 200 224; do for g in 1 2; do
  TW_K2_RING_KB=$ring TW_K2_GROUPS=$g K2_SIZES=512,1024,1536,2048,4096 timeout 300 python tools/k2_small_t.py > $o/k2_ring${ring}_g${g}.txt 2>&1
done; done
echo done
