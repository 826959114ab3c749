# One command for an N-GPU NVSwitch box (the evidence this round could not
# produce on one-GPU boxes).  Everything lands in gpurun_out/mgpu/.
#   bash tools/validate_multigpu.sh [N]
set -x
N=${1:-$(python -c "import torch; print(min(torch.cuda.device_count(), 8))")}
OUT=gpurun_out/mgpu
mkdir -p $OUT
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
# 1. NVLS K1 parity against the oracle (single process, N devices) + the full GPU suite
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python -m pytest tests/test_k1_gpu.py -q -m gpu -k nvls_multi_gpu > $OUT/nvls_parity.log 2>&1; tail -2 $OUT/nvls_parity.log
timeout 1800 python -m pytest tests/test_nvls_gpu.py -q -m gpu -k nvls_hw -rs > $OUT/nvls_hw.log 2>&1; tail -4 $OUT/nvls_hw.log
# 2. bench.py at N = 2, 4, ..., N (the driver's scaling run), both arms
for n in 2 4 8; do
  [ $n -le $N ] || continue

  $RUN $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n > $OUT/bench_tp$n.json 2> $OUT/bench_tp$n.err
  $RUN $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --impl reference > $OUT/bench_ref_tp$n.json 2>/dev/null
  $RUN $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --gather-residual > $OUT/bench_tp${n}_g2.json 2>/dev/null
done
# 3. configs[2]/[4]: token x SM-budget sweep with the K3+K2 and NCCL+K2 baselines
$RUN $N --master-addr 127.0.0.1 --master-port 29640 tools/sweep_tp.py --out $OUT/sweep_tp$N.json > $OUT/sweep.log 2>&1
# 4. the weave with K1 as the boundary op (Llama / Mixtral), and serving throughput
$RUN $N --master-addr 127.0.0.1 --master-port 29641 tools/weave_bench.py --out $OUT/weave_tp$N.json > $OUT/weave.log 2>&1
$RUN $N --master-addr 127.0.0.1 --master-port 29642 tools/throughput_bench.py --out $OUT/throughput_tp$N.json > $OUT/throughput.log 2>&1
# 5. NVLink payload bytes around the TP leg (driver counters, no replay)
bash tools/profile_tp.sh $N > $OUT/nvlink.txt 2>&1
cp gpurun_out/nvlink_*.txt $OUT/ 2>/dev/null
echo done
