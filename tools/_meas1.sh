set -x
o=gpurun_out/m1
mkdir -p $o
timeout 400 python bench.py > $o/bench.json 2> $o/bench.err
timeout 200 python bench.py --impl reference --steps 5 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err
timeout 300 python tools/k2_small_t.py > $o/k2_small_t.txt 2>&1
timeout 300 python tools/k1_small.py > $o/k1_small_dev.txt 2>&1
TW_FORCE_SYS_SCOPE=1 timeout 300 python tools/k1_small.py > $o/k1_small_sys.txt 2>&1
timeout 300 python tools/k1_small.py --transport nvls_sim > $o/k1_small_nvlssim.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2 -s 3 -c 1 -o $o/k2_t1024 -f python tools/k2_small_t.py profile 1024 > $o/ncu1024.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2 -s 3 -c 1 -o $o/k2_t8192 -f python tools/k2_small_t.py profile 8192 > $o/ncu8192.log 2>&1
echo done
