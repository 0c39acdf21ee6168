# 4-GPU round check: multi-GPU tests, N=2/4 bench lines, in-process NVLink
# kernel timings and ncu NVLink/DRAM counters per multi-GPU kernel.
O=gpurun_out/g4; mkdir -p $O/ncu
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
for n in 2 4; do for p in all-reduce pull-gossip elastic-avg push-gossip; do
  timeout 120 python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 30 >> $O/inproc_wall.jsonl 2>> $O/inproc_wall.err
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
for n in 2 4; do for p in all-reduce pull-gossip elastic-avg; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu/nvl_${p}_n${n}.csv \
    python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 2 --warmup 1 > $O/ncu/nvl_${p}_n${n}.log 2>&1
  echo ncu_${p}_n${n}=$? >> $O/status.txt
done; done
