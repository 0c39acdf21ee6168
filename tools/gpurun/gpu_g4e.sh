# 4-GPU: binding fix check, NCCL library baseline, bench N=2/4, ncu NVLink counters
O=gpurun_out/g4e; mkdir -p $O/ncu
timeout 600 python -m pytest tests/test_reference_binding.py tests/test_inproc_ranks.py -q -rf > $O/bind_inproc.log 2>&1; echo bind_inproc=$? >> $O/status.txt
for n in 2 4; do for algo in auto NVLS Ring; do
  if [ $algo = auto ]; then unset NCCL_ALGO; else export NCCL_ALGO=$algo; fi
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/nccl_allreduce_probe.py >> $O/nccl_probe.jsonl 2>> $O/nccl_probe.err
  echo nccl_${algo}_n$n=$? >> $O/status.txt
done; done
unset NCCL_ALGO
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
for n in 4 2; do for p in all-reduce pull-gossip elastic-avg; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu/nvl_${p}_n${n}.csv \
    python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 2 --warmup 1 > $O/ncu/nvl_${p}_n${n}.log 2>&1
  echo ncu_${p}_n${n}=$? >> $O/status.txt
done; done
