# Re-measure what profiles/ quotes (one GPU).  Outputs land in gpurun_out/rNN/;
# the ones kept are copied to profiles/ with the round suffix.
#   bash tools/refresh_profiles.sh r02
set -x
R=${1:-r02}
out=gpurun_out/$R
mkdir -p $out
nvidia-smi -q > $out/nvidia_smi_q.txt 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err
# the N>1 leg's plumbing: two ranks co-located on this one GPU (PEER; not NVLink)
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --tokens 2048 > $out/bench_tp2_colocated.json 2> $out/bench_tp2.err
# launch list of the bench command (per-launch device times, cold and serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $out/launches.csv \
  python bench.py --steps 5 --warmup 3 --quick > /dev/null 2>&1
# one full capture of the dominant kernel (K2 at 8192 x 8192) and of K2 at T = 1024
ncu --set full --clock-control none --import-source on -k regex:k2_tma -s 3 -c 1 -o $out/k2_full -f \
  python bench.py --steps 2 --warmup 3 --quick > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2 -s 2 -c 1 -o $out/k2_t1024 -f \
  python tools/k2_small_t.py profile 1024 > /dev/null 2>&1
# the north_star kernel's code path on simulated ranks (NVLS_SIM, TP = 8, T = 1024) and K1 PEER
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o $out/k1_nvls_sim_w8 -f \
  python tools/k1_profile.py 8 1024 nvls_sim > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 -o $out/k1_peer_w8 -f \
  python tools/k1_profile.py 8 8192 peer > /dev/null 2>&1
# decode-size latency of the fused op (barrier cost) at each barrier scope / transport
timeout 300 python tools/k1_small.py --out $out/k1_small_dev.json > /dev/null 2>&1
TW_FORCE_SYS_SCOPE=1 timeout 300 python tools/k1_small.py --out $out/k1_small_sys.json > /dev/null 2>&1
timeout 300 python tools/k1_small.py --transport nvls_sim --out $out/k1_small_nvls_sim.json > /dev/null 2>&1
timeout 900 python tools/tp_colocated_sweep.py --out $out/tp_colocated.json > $out/tp_colocated.log 2>&1
# (compute-sanitizer runs: tools/sanitize_all.sh -> profiles/sanitizer_r02.txt; the tool has
# since been closed on the GPU pool, so the refresh no longer calls it)
# summaries on the box (gpurun brings back <= 64 MiB): keep one full report
A8192=$((4 * 8192 * 8192 * 2 + 4 * 8192))
A1024=$((4 * 1024 * 8192 * 2 + 4 * 8192))
python tools/ncu_summary.py $out/k2_full.ncu-rep --alg-bytes $A8192 --command "ncu --set full -k regex:k2_tma -s 3 -c 1 python bench.py --steps 2 --warmup 3 --quick" > $out/k2_ncu.json
python tools/ncu_summary.py $out/k2_t1024.ncu-rep --alg-bytes $A1024 --command "ncu --set full -k regex:k2 -s 2 -c 1 python tools/k2_small_t.py profile 1024" > $out/k2_t1024_ncu.json
python tools/ncu_summary.py $out/k1_nvls_sim_w8.ncu-rep --command "ncu --set full -k regex:k1_ -s 2 -c 1 python tools/k1_profile.py 8 1024 nvls_sim" --note "8 simulated ranks on ONE GPU (MmSim: per-rank loads/stores in place of multimem); HBM-bound stand-in of the NVLS kernel" > $out/k1_nvls_sim_w8_ncu.json
python tools/ncu_summary.py $out/k1_peer_w8.ncu-rep --command "ncu --set full -k regex:k1_ -s 2 -c 1 python tools/k1_profile.py 8 8192 peer" > $out/k1_peer_w8_ncu.json
rm -f $out/k2_t1024.ncu-rep $out/k1_peer_w8.ncu-rep $out/k1_nvls_sim_w8.ncu-rep
ls -la $out
echo done
