# 4-GPU follow-up: binding failure bisection, in-process NVLink walls, ncu NVLink counters
O=gpurun_out/g4b; mkdir -p $O/ncu
timeout 300 python -m pytest tests/test_reference_binding.py -q -x -rf > $O/bind_alone.log 2>&1; echo bind_alone=$? >> $O/status.txt
timeout 900 python -m pytest tests/test_multigpu.py tests/test_reference_binding.py -q -rf > $O/bind_after_mgpu.log 2>&1; echo bind_after_mgpu=$? >> $O/status.txt
for n in 2 4; do for p in all-reduce pull-gossip elastic-avg push-gossip; do
  timeout 120 python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 30 >> $O/inproc_wall.jsonl 2>> $O/inproc_wall.err
  echo wall_${p}_n${n}=$? >> $O/status.txt
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
for n in 2 4; do for p in all-reduce pull-gossip elastic-avg; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu/nvl_${p}_n${n}.csv \
    python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 2 --warmup 1 > $O/ncu/nvl_${p}_n${n}.log 2>&1
  echo ncu_${p}_n${n}=$? >> $O/status.txt
done; done
