# 4-GPU: full multi-GPU suite, N=4 bench (staged EASGD chain), NCCL NVLS baseline, ncu NVLink at N=4
O=gpurun_out/${OUT:-g4f}; mkdir -p $O/ncu
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_inproc_ranks.py tests/test_reference_binding.py -q -rf > $O/pytest_mgpu.log 2>&1; echo pytest_mgpu=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 --no-cpu > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
for algo in NVLS NVLSTree auto; do
  if [ $algo = auto ]; then unset NCCL_ALGO; else export NCCL_ALGO=$algo; fi
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 tools/nccl_allreduce_probe.py --op sum >> $O/nccl_probe.jsonl 2>> $O/nccl_probe.err
  echo nccl_${algo}=$? >> $O/status.txt
done
unset NCCL_ALGO
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
for p in pull-gossip elastic-avg all-reduce; do
  DSGD_ALLREDUCE=p2p timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu/nvl_${p}_n4_p2p.csv \
    python tools/nvlink_profile.py --gpus 4 --protocol $p --rounds 2 --warmup 1 > $O/ncu/nvl_${p}_n4_p2p.log 2>&1
  echo ncu_${p}_n4=$? >> $O/status.txt
done
timeout 900 ncu --replay-mode application --metrics $M --clock-control none --csv --log-file $O/ncu/nvl_all-reduce_n4_nvls.csv \
    python tools/nvlink_profile.py --gpus 4 --protocol all-reduce --rounds 2 --warmup 1 > $O/ncu/nvl_all-reduce_n4_nvls.log 2>&1
echo ncu_nvls_app=$? >> $O/status.txt
