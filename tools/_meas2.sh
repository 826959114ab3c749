set -x
o=gpurun_out/m2
mkdir -p $o
timeout 900 python -m pytest tests/test_k2_gpu.py tests/test_dropin.py -m gpu -q -p no:cacheprovider -k "host or dropin or Dropin" > $o/tests.txt 2>&1
tail -3 $o/tests.txt
./build/bench/dropin_bench rmsnorm 8192 8192 2 5 > $o/dropin.json 2>&1
./build/bench/dropin_bench fused 8 1024 8192 1 3 > $o/dropin_fused.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2 -s 2 -c 1 -o $o/k2_t1024 -f python tools/k2_small_t.py profile 1024 > $o/ncu1024.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2 -s 2 -c 1 -o $o/k2_t8192 -f python tools/k2_small_t.py profile 8192 > $o/ncu8192.log 2>&1
nproc > $o/nproc.txt; lscpu > $o/lscpu.txt; numactl -H > $o/numa.txt 2>&1; nvidia-smi topo -m > $o/topo.txt 2>&1
echo done
