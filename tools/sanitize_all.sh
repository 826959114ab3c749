# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py,
# TMA engine with one and two row groups and the default policy.
set -x
out=gpurun_out/san
mkdir -p $out
for g in 1 2; do
 for tool in memcheck racecheck synccheck; do
  TW_K2_ENGINE=tma TW_K2_GROUPS=$g timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > $out/sanitize_${tool}_tma_g$g.log 2>&1
 done
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > $out/sanitize_${tool}_default.log 2>&1
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY" $out/*.log
