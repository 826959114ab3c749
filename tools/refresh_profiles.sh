# Re-measure everything profiles/ quotes for the bench line and the TP=1 sweeps
# (one GPU).  Outputs land in gpurun_out/; copy the ones you keep to profiles/.
set -x
out=gpurun_out
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $out/launches.csv \
  python bench.py --steps 5 --warmup 3 --quick > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_tma -s 3 -c 1 -o $out/k2_full -f \
  python bench.py --steps 2 --warmup 3 --quick > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_tma -s 2 -c 1 -o $out/k2_budget16 -f \
  python tools/k2_budget_profile.py 16 > /dev/null 2>&1
timeout 900 python tools/sweep.py --out $out/sweep.json > $out/sweep.log 2>&1
timeout 900 python tools/export_calibration.py --out $out/microbench_b200_measured.json > $out/export.log 2>&1
python tools/k2_policy_check.py > $out/k2_policy.json 2> $out/k2_policy.err
echo done
