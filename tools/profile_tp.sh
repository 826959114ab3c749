# For an N-GPU box (not runnable on a one-GPU box): NVLink bytes, DRAM bytes
# and device time of the fused op K1 on rank 0, per launch, while every rank
# runs bench.py's TP leg.  Metric names from `ncu --query-metrics --chip gb100`
# on this pod (profiles/ncu_nvlink_metrics_b200.txt).  ncu serialises and
# replays the kernel, so only the BYTES are meaningful here, not the time;
# per-direction NVLink GB/s = nvltx__bytes (egress) / nvlrx__bytes (ingress)
# over bench.py's own device time.
N=${1:-8}
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
  tools/ncu_rank0.py \
  ncu --target-processes all --clock-control none -k regex:rownorm_kernel -c 3 \
      --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
      --csv --log-file gpurun_out/k1_nvlink_rank0.csv \
  -- python bench.py --gpus $N --steps 3 --warmup 3
