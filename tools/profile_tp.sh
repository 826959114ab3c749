# For an N-GPU NVSwitch box (not runnable on a one-GPU box): NVLink bytes moved
# by bench.py's TP leg, from the driver's per-link throughput counters
# (`nvidia-smi nvlink -gt d`, TX/RX data payload in KiB) sampled before and
# after the run -- no kernel replay (ncu replays a kernel once per metric
# pass, and a replayed K1 waits forever on peers that are not replayed; a
# two-process trial on one GPU hung that way).  Divide by bench.py's own
# device time (max over ranks) for NVLink GB/s per GPU per direction, to set
# against B = S*(G + 1/N) and 900 GB/s.
N=${1:-8}
STEPS=${2:-20}
mkdir -p gpurun_out
nvidia-smi nvlink -gt d > gpurun_out/nvlink_before.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus $N --steps $STEPS --warmup 3 > gpurun_out/bench_tp$N.json
nvidia-smi nvlink -gt d > gpurun_out/nvlink_after.txt
python tools/nvlink_delta.py gpurun_out/nvlink_before.txt gpurun_out/nvlink_after.txt
