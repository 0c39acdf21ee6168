# 2-GPU: staged EASGD chain publish-batch sweep (in-process wall + distributed bench)
O=gpurun_out/${OUT:-g2d}; mkdir -p $O
for pb in 1 2 4 8 16 32; do
  DSGD_EA_PUBLISH=$pb timeout 120 python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 30 | sed "s/^{/{\"publish\": $pb, /" >> $O/wall.jsonl 2>> $O/wall.err
done
for pb in 2 4 8 16; do
  DSGD_EA_PUBLISH=$pb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + pb)) bench.py --gpus 2 --no-cpu > $O/bench_n2_pub$pb.json 2> $O/bench_n2_pub$pb.err
done
