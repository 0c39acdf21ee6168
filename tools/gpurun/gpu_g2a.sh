# 2-GPU: staged EASGD chain -- parity (in-process + distributed), wall, bench, ncu
O=gpurun_out/${OUT:-g2a}; mkdir -p $O
timeout 600 python -m pytest tests/test_inproc_ranks.py -q -rf -x -k "elastic" > $O/inproc_ea.log 2>&1; echo inproc_ea=$? >> $O/status.txt
timeout 900 python -m pytest tests/test_multigpu.py -q -rf -x -k "protocols and default" > $O/mgpu_default.log 2>&1; echo mgpu=$? >> $O/status.txt
for st in 1 0; do
  DSGD_EA_STAGED=$st timeout 120 python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 30 >> $O/wall.jsonl 2>> $O/wall.err
  echo wall_staged$st=$? >> $O/status.txt
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
DSGD_EA_STAGED=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 2 > $O/bench_n2_old.json 2> $O/bench_n2_old.err; echo n2_old=$? >> $O/status.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/nvl_ea_n2.csv python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 2 --warmup 1 > $O/nvl_ea_n2.log 2>&1; echo ncu=$? >> $O/status.txt
